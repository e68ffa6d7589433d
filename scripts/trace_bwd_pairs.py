"""Per-pair timeline of CTA 0 in a bwd trace build (UB_LIB=.../libub_trace.so):
compute warp 0: 1 pair start, 2 Q/dO tile and S seen, 3 exp done, 4 P~ handed over, 5 dP seen,
7 dS handed over; MMA warp 13: 12 P~ seen (dV issue), 10 S_{p+1} issued, 19 dQ issued.
Prints per-pair durations (cycles) and their means."""
import ctypes as C, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2208_08124_b200 as ub
from paper_2208_08124_b200 import _lib
import synth
from gpu_util import make_batch
pd = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
L = synth.gen_lengths("mlperf_like_v0", 56, 0)
lengths, off, qkv, dout = make_batch(L, 16, 64)
cu = torch.tensor(off.astype(np.int32)).cuda(); qd = qkv.cuda(); gd = dout.cuda()
o, lse = ub.varlen_fmha_fwd(qd, cu, 512, p_dropout=pd)
for _ in range(3): ub.varlen_fmha_bwd(qd, o, lse, gd, cu, 512, p_dropout=pd)
torch.cuda.synchronize()
buf = np.zeros(16 * 1024, dtype=np.uint64)
f = _lib.lib().ub_debug_bwd_trace; f.restype = C.c_int; f.argtypes = [C.c_void_p, C.c_size_t]
assert f(buf.ctypes.data_as(C.c_void_p), buf.nbytes) == 0
ev = (buf >> np.uint64(48)).astype(np.int64); ck = (buf & np.uint64(0xFFFFFFFFFFFF)).astype(np.int64)
t0 = ck[ck > 0].min()
def ser(w, e):
    return np.array([int(ck[w * 1024 + i] - t0) for i in range(1024) if buf[w * 1024 + i] and ev[w * 1024 + i] == e])
c = {e: ser(0, e) for e in (1, 2, 3, 4, 5, 7)}
c4 = {e: ser(4, e) for e in (1, 2, 3, 4, 5, 7)}
m = {e: ser(13, e) for e in (12, 10, 19)}
n = min(len(v) for v in list(c.values()) + list(m.values())) - 1
cols = {
    "in_wait": c[2][:n] - c[1][:n], "exp": c[3][:n] - c[2][:n],
    "p_store": c[4][:n] - c[3][:n], "dp_wait": c[5][:n] - c[4][:n], "B": c[7][:n] - c[5][:n],
    "gap": c[1][1:n + 1] - c[7][:n], "pair": c[1][1:n + 1] - c[1][:n],
    "P->mma": m[12][:n] - c[4][:n], "mmaS->seen": c[2][1:n + 1] - m[10][:n],
    "dS->dQiss": m[19][:n] - c[7][:n], "wg1_lag": c4[4][:n] - c[4][:n],
}
print(f"p={pd} pairs traced {n}; CTA0 span {ck.max() - t0}")
print("pair " + " ".join(f"{k:>10s}" for k in cols))
for i in range(min(n, 48)):
    print(f"{i:4d} " + " ".join(f"{int(v[i]):10d}" for v in cols.values()))
print("mean " + " ".join(f"{v.mean():10.0f}" for v in cols.values()))
print("med  " + " ".join(f"{np.median(v):10.0f}" for v in cols.values()))
