"""Dev probe: host (CPU) cost of enqueuing each hot-path call, in microseconds.
Python binding vs the bare C call with pre-marshalled arguments."""
import sys, time, ctypes as C
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2208_08124_b200 as ub
from paper_2208_08124_b200 import api
import synth
from gpu_util import make_batch

L = synth.gen_lengths("mlperf_like_v0", 56, 0)
lengths, off, qkv, dout = make_batch(L, 16, 64)
cu = torch.tensor(off.astype(np.int32)).cuda(); qd = qkv.cuda(); gd = dout.cuda()
o, lse = ub.varlen_fmha_fwd(qd, cu, 512)
dq = ub.varlen_fmha_bwd(qd, o, lse, gd, cu, 512)
padded = torch.empty((56, 512, 16, 64), dtype=torch.bfloat16, device="cuda")
torch.cuda.synchronize()


def host(fn, n=60):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    return 1e6 * float(np.median(ts))


lib = api.lib()
prm = api.fmha_params(56, qd.shape[0], 512, 16, 64, torch.bfloat16)
ws_f = api._workspace(lib.ub_fmha_workspace_bytes(C.byref(prm), 0), qd.device, "fmha_fwd")
ws_b = api._workspace(lib.ub_fmha_workspace_bytes(C.byref(prm), 1), qd.device, "fmha_bwd")
s = api._stream(None)
args_f = (C.byref(prm), api._ptr(qd), api._ptr(cu), api._ptr(o), api._ptr(lse), api._ptr(ws_f), s)
args_b = (C.byref(prm), api._ptr(qd), api._ptr(o), api._ptr(lse), api._ptr(gd), api._ptr(cu), api._ptr(dq),
          api._ptr(ws_b), s)
r = {
    "fwd_py": host(lambda: ub.varlen_fmha_fwd(qd, cu, 512, out=o, lse=lse)),
    "fwd_c": host(lambda: lib.ub_varlen_fmha_fwd(*args_f)),
    "bwd_py": host(lambda: ub.varlen_fmha_bwd(qd, o, lse, gd, cu, 512, dqkv=dq)),
    "bwd_c": host(lambda: lib.ub_varlen_fmha_bwd(*args_b)),
    "pad_py": host(lambda: ub.pad(o, cu, 56, 512, out=padded)),
    "slice": host(lambda: qd[:1000]),
    "stream": host(lambda: api._stream(None)),
    "params": host(lambda: api.fmha_params(56, 14000, 512, 16, 64, torch.bfloat16)),
    "ptr": host(lambda: api._ptr(qd)),
}
print(" ".join(f"{k}={v:.1f}us" for k, v in r.items()))
