"""Per-tile check of the symmetric kernel's raw transposed products D_T (debug
dump): for each (pair a, column tile c >= 2a + 2, CTA r), D_T = P_r^T V_{2a+r}
scaled.  usage: NCGP_SYM_ITEM=L python tools/sym_diag3.py n"""
import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2310_20285_b200 import _native
from paper_2310_20285_b200.kernels import KernelOperator
torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
d, w, WP = 8, 32, 32
rng = np.random.default_rng(1)
X = rng.standard_normal((n, d)); V = rng.standard_normal((n, w))
Xf = torch.from_numpy(X).float().cuda(); Vf = torch.from_numpy(V).float().cuda()
op = KernelOperator("rbf", 1.5, 1.0, Xf, w_max=32)
nb = (n + 127) // 128
pairs = ((nb + 1) // 2 * 2) // 2
dump = torch.full((pairs, nb, 2, 128, WP), float("nan"), device="cuda")
lib = _native.load()
lib.ncgp_debug_set_sym_dump.argtypes = [ctypes.c_void_p]
lib.ncgp_debug_set_sym_dump(ctypes.c_void_p(dump.data_ptr()))
os.environ["NCGP_SYM"] = "1"
op.apply(Vf); torch.cuda.synchronize()
lib.ncgp_debug_set_sym_dump(ctypes.c_void_p(0))
D = dump.cpu().numpy()
# reference: K(X_c, X_rows(2a+r)) V_rows(2a+r), up to the power-of-two scale (compare normalised)
X64 = torch.from_numpy(X).cuda(); V64 = torch.from_numpy(V).cuda()
bad = []
for a in range(pairs):
    for c in range(2 * a + 2, nb):
        for r in range(2):
            rt = 2 * a + r
            if rt >= nb: continue
            rows = slice(128 * rt, min(n, 128 * rt + 128))
            cols = slice(128 * c, min(n, 128 * c + 128))
            ref = KernelOperator("rbf", 1.5, 1.0, X64[cols], X64[rows], w_max=32).apply(V64[rows]).cpu().numpy()
            got = D[a, c, r, : ref.shape[0], :w].astype(np.float64)
            # each RHS column carries its own power-of-two scale: fit it per column
            sc = np.where(np.abs(ref).sum(0) > 0,
                          2.0 ** np.round(np.log2(np.maximum(np.abs(got).sum(0), 1e-300) /
                                                  np.maximum(np.abs(ref).sum(0), 1e-300))), 1.0)
            e = np.abs(got / sc - ref).max() / max(np.abs(ref).max(), 1e-30)
            if not np.isfinite(e) or e > 1e-3:
                bad.append((a, c, r, float(e)))
print("item", os.environ.get("NCGP_SYM_ITEM", "128"), "bad (a, c, rank, err):", bad[:20], len(bad))

# which V block does a bad dump use?  D_T(a, c, r) = K(X_c, X_rt) V_rt; try V_x
for (a, c, r, e) in bad[:4]:
    rt = 2 * a + r
    rows = slice(128 * rt, min(n, 128 * rt + 128))
    cols = slice(128 * c, min(n, 128 * c + 128))
    Kc = KernelOperator("rbf", 1.5, 1.0, X64[cols], X64[rows], w_max=128)
    got = D[a, c, r, : cols.stop - cols.start, :w].astype(np.float64)
    best = []
    for x in range(nb):
        vx = V64[128 * x: 128 * x + (rows.stop - rows.start)]
        if vx.shape[0] != rows.stop - rows.start: continue
        ref = Kc.apply(vx.contiguous()).cpu().numpy()
        sc = np.where(np.abs(ref).sum(0) > 0, 2.0 ** np.round(np.log2(np.maximum(np.abs(got).sum(0), 1e-300) / np.maximum(np.abs(ref).sum(0), 1e-300))), 1.0)
        best.append((float(np.abs(got / sc - ref).max() / max(np.abs(ref).max(), 1e-30)), x))
    best.sort()
    print(f"  dump (a={a}, c={c}, r={r}): best V blocks {best[:3]}")
