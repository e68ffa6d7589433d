"""Correlate the warps of CTA 0 in a bwd trace build, per iteration / pair j (cycles from kernel
start): producer stage wait passed (23) / arrived (24); MMA: S_{j+1}, dP_j issued (10), P~_j seen
(12), dS_{j-1} seen (13), dK/dQ issued (19); compute warp 0: iteration start (1), S_j / dP_{j-1}
waits passed (2), P~_j stored (4), dS_{j-1} stored (7); epilogue warp 8: dQ in (31), out (32)."""
import ctypes as C, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2208_08124_b200 as ub
from paper_2208_08124_b200 import _lib
import synth
from gpu_util import make_batch
L = synth.gen_lengths("mlperf_like_v0", 56, 0)
lengths, off, qkv, dout = make_batch(L, 16, 64)
cu = torch.tensor(off.astype(np.int32)).cuda(); qd = qkv.cuda(); gd = dout.cuda()
o, lse = ub.varlen_fmha_fwd(qd, cu, 512)
for _ in range(3): ub.varlen_fmha_bwd(qd, o, lse, gd, cu, 512)
torch.cuda.synchronize()
buf = np.zeros(16 * 1024, dtype=np.uint64)
f = _lib.lib().ub_debug_bwd_trace; f.restype = C.c_int; f.argtypes = [C.c_void_p, C.c_size_t]
assert f(buf.ctypes.data_as(C.c_void_p), buf.nbytes) == 0
ev = (buf >> np.uint64(48)).astype(np.int64); ck = (buf & np.uint64(0xFFFFFFFFFFFF)).astype(np.int64)
t0 = ck[ck > 0].min()
def series(w, e):
    return [int(ck[w * 1024 + i] - t0) for i in range(1024) if buf[w * 1024 + i] and ev[w * 1024 + i] == e]
cols = [("pSt", 12, 23), ("pArr", 12, 24), ("mSdP", 13, 10), ("mdV", 13, 12), ("mdKQ", 13, 13), ("mGrd", 13, 19),
        ("c1", 0, 1), ("cIn", 0, 2), ("cP", 0, 4), ("cdS", 0, 7),
        ("eQin", 8, 31), ("eKV", 8, 33), ("eQfree", 8, 34), ("eQout", 8, 32)]
ser = {n: series(w, e) for n, w, e in cols}
print("pair " + " ".join(f"{n:>7s}" for n, _, _ in cols))
for p in range(min(40, len(ser["cIn"]))):
    print(f"{p:4d} " + " ".join(f"{(ser[n][p] if p < len(ser[n]) else -1):7d}" for n, _, _ in cols))
