"""Timeline of CTA 0 of the bwd kernel (trace build)."""
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
for _ in range(3): d = ub.varlen_fmha_bwd(qd, o, lse, gd, cu, 512)
torch.cuda.synchronize()
buf = np.zeros(16 * 1024, dtype=np.uint64)
f = _lib.lib().ub_debug_bwd_trace; f.restype = C.c_int; f.argtypes = [C.c_void_p, C.c_size_t]
assert f(buf.ctypes.data_as(C.c_void_p), buf.nbytes) == 0
ev = (buf >> np.uint64(48)).astype(np.int64); ck = (buf & np.uint64(0xFFFFFFFFFFFF)).astype(np.int64)
t0 = ck[ck > 0].min()
names = {11: "S_issued", 19: "grads_issued", 24: "P_lse_st", 1: "c_wait", 2: "S_got", 3: "ld_done", 4: "cmp_done", 5: "pds_empty_ok", 6: "dq_epi_done", 7: "pds_full", 8: "dkv_wait", 9: "dkv_ok",
         10: "S_issue", 12: "grads_issue", 16: "item", 17: "kv_ok", 18: "qdo_ok", 20: "P_item", 21: "P_kv_ok", 22: "P_q", 23: "P_q_ok",
         30: "E_dq_wait", 31: "E_dq_ok", 32: "E_dq_out", 33: "E_dkv_wait", 34: "E_dkv_ok"}
for w in (0, 4, 8, 12, 13, 14):
    print(f"--- warp {w}")
    row = [(ev[w * 1024 + i], ck[w * 1024 + i] - t0) for i in range(1024) if buf[w * 1024 + i]]
    prev = None; out = []
    for e, c in row[:80]:
        out.append(f"{names.get(int(e), e)}@{c}" + (f"(+{c - prev})" if prev is not None else "")); prev = c
    print(" ".join(out))
