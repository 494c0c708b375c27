"""A/B timing of K1-sym1 builds and debug ablations (wrong results for the
ablations).  usage: python tools/sym_ab.py [n] [family] [w]
Runs each library in tools/ab/*.so plus the in-tree build in a subprocess."""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json, ctypes
import numpy as np, torch
sys.path.insert(0, %r)
from paper_2310_20285_b200 import _native as N
from paper_2310_20285_b200.kernels import KernelOperator
n, fam, w = %d, %r, %d
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, 8))).float().cuda()
V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
os.environ["NCGP_SYM"] = "1"; os.environ["NCGP_SYM_CG"] = "1"
op = KernelOperator(fam, 1.5, 1.0, X, w_max=32)
lib = N.load()
res = {}
trace = torch.zeros(1 << 20, dtype=torch.int64, device="cuda")
for dbg in %r:
    if dbg is not None:
        os.environ["NCGP_SYM_DBG"] = str(dbg)
        lib.ncgp_debug_set_trace.argtypes = [ctypes.c_void_p]
        lib.ncgp_debug_set_trace(trace.data_ptr())
    op.apply(V); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        op.apply(V)
    e1.record(); torch.cuda.synchronize()
    res[str(dbg)] = round(e0.elapsed_time(e1) / 5, 3)
    if dbg is not None:
        lib.ncgp_debug_set_trace(None)
print(json.dumps(res))
'''


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
    fam = sys.argv[2] if len(sys.argv) > 2 else "rbf"
    w = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    libs = [("in-tree", None)] + [(os.path.basename(p), p) for p in sorted(glob.glob(os.path.join(ROOT, "tools", "ab", "*.so")))]
    for name, path in libs:
        dbgs = [None, 1, 2, 3, 8] if path is None else [None]
        env = dict(os.environ)
        if path:
            env["NCGP_LIB"] = path
        out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, n, fam, w, dbgs)], env=env,
                             capture_output=True, text=True, timeout=600)
        print(name, out.stdout.strip() or out.stderr[-800:], flush=True)


if __name__ == "__main__":
    main()
