"""Build the CPU oracle library (test infrastructure only -- see oracle.c).

Tries gcc with OpenMP first (the CPU baseline uses all host threads), then
falls back to a single-threaded build.  Output: oracle/liboracle.so.
"""
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.c")
LIB = os.path.join(HERE, "liboracle.so")


def _compilers():
    seen = []
    for cc in ("/usr/bin/gcc", os.environ.get("CC"), "gcc", "cc"):
        if cc and cc not in seen and (os.path.isabs(cc) and os.path.exists(cc) or shutil.which(cc)):
            seen.append(cc)
    return seen


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    base = ["-O2", "-fPIC", "-shared", "-ffp-contract=off", "-std=gnu11", "-Wall"]
    errors = []
    for cc in _compilers():
        for extra in (["-fopenmp"], []):
            cmd = [cc, *base, *extra, "-o", LIB + ".tmp", SRC, "-lm"]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode == 0:
                os.replace(LIB + ".tmp", LIB)
                return LIB
            errors.append(" ".join(cmd) + "\n" + r.stderr)
    raise RuntimeError("could not build the oracle:\n" + "\n".join(errors))


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
