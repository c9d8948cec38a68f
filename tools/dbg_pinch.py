import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, torch
from conftest import load_case
from paper_2204_05438_b200 import distributed as D
tri, g = load_case('aniso2k_s1')
n, T = tri.n_vertices, tri.n_triangles
dev = torch.device('cuda',0)
xy = torch.from_numpy(tri.vertices).to(dev); tr = torch.from_numpy(tri.triangles).to(dev)
for world in (1, 2):
    for b, e in D.partition(T, world):
        try:
            off, v, p, f, st = D.run_partition(xy, tr, n, T, b, e)
            print(world, b, e, p, f, st)
        except Exception as ex:
            print(world, b, e, 'ERR', ex)
print('golden stats', g['stats'])
