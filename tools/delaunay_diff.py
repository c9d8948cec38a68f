"""Where the GPU Delaunay and Qhull disagree: the differing triangles and an
exact (rational) Delaunay test of the disputed diagonals."""
import os
import sys
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2204_05438_b200.delaunay import delaunay_gpu  # noqa: E402


def incircle_exact(a, b, c, d):
    A = [Fraction(x) for x in a]; B = [Fraction(x) for x in b]; C = [Fraction(x) for x in c]; D = [Fraction(x) for x in d]
    adx, ady = A[0] - D[0], A[1] - D[1]
    bdx, bdy = B[0] - D[0], B[1] - D[1]
    cdx, cdy = C[0] - D[0], C[1] - D[1]
    det = (adx * adx + ady * ady) * (bdx * cdy - cdx * bdy) + (bdx * bdx + bdy * bdy) * (cdx * ady - adx * cdy) + \
        (cdx * cdx + cdy * cdy) * (adx * bdy - bdx * ady)
    return (det > 0) - (det < 0)


def orient_exact(a, b, c):
    A = [Fraction(x) for x in a]; B = [Fraction(x) for x in b]; C = [Fraction(x) for x in c]
    d = (B[0] - A[0]) * (C[1] - A[1]) - (B[1] - A[1]) * (C[0] - A[0])
    return (d > 0) - (d < 0)


def main():
    from scipy.spatial import Delaunay
    n, seed = int(sys.argv[1]), int(sys.argv[2])
    pts = np.random.default_rng(seed).uniform((0.0, 0.0), (1.0, 1.0), (n, 2))
    t, info = delaunay_gpu(pts)
    q = Delaunay(pts).simplices.astype(np.int64)
    key = lambda r: tuple(sorted(int(x) for x in r))  # noqa: E731
    sg = set(map(key, t))
    sq = set(map(key, q))
    only_g, only_q = sg - sq, sq - sg
    print("n", n, "seed", seed, "gpu-only", len(only_g), "qhull-only", len(only_q), flush=True)

    def bad_triangles(tris):
        # a triangle is non-Delaunay if some vertex of an adjacent differing triangle lies inside it (exactly)
        out = 0
        pool = set(v for tr in tris for v in tr)
        for tr in list(tris)[:50]:
            a, b, c = (pts[i] for i in tr)
            if orient_exact(a, b, c) < 0:
                b, c = c, b
            for v in pool:
                if v in tr:
                    continue
                if incircle_exact(a, b, c, pts[v]) > 0:
                    out += 1
                    print("  not Delaunay:", tr, "contains", v, flush=True)
                    break
        return out

    print("gpu-only triangles violating exactly:", bad_triangles(only_g))
    print("qhull-only triangles violating exactly:", bad_triangles(only_q))


if __name__ == "__main__":
    main()
