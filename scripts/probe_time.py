"""Dev probe: fwd/bwd timing at BERT-large config 2 (not a bench number).
Reports the whole call and the main kernel alone (library profile events)."""
import sys
import os; _R = os.environ.get("UB_ROOT", "/root/repo"); sys.path.insert(0, _R); sys.path.insert(0, _R + "/tests")
import numpy as np, torch
import paper_2208_08124_b200 as ub
from paper_2208_08124_b200 import api as _api
ub.dropout_mask = _api.dropout_mask
import synth
from gpu_util import make_batch
dist = sys.argv[1] if len(sys.argv) > 1 else "mlperf_like_v0"
p = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
L = synth.gen_lengths(dist, 56, 0)
lengths, off, qkv, dout = make_batch(L, 16, 64)
cu = torch.tensor(off.astype(np.int32)).cuda(); qd = qkv.cuda(); gd = dout.cuda()
T = int(off[-1]); s2 = float((L.astype(np.int64)**2).sum())
def t(fn, kid, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(n)]
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for i in range(n):
        ub.api.profile_events(kid, *evs[i]); fn()
    e1.record(); torch.cuda.synchronize()
    ub.api.profile_events(kid)
    return e0.elapsed_time(e1) / n * 1e3, np.median([a.elapsed_time(b) for a, b in evs]) * 1e3
# MASK=1 (default for p > 0): the step's materialised keep bits, as the bench step uses them
mk = ub.dropout_mask(cu, T, 16, 512, p) if p > 0 and os.environ.get("MASK", "1") == "1" else None
o, lse = ub.varlen_fmha_fwd(qd, cu, 512, p_dropout=p, dropout_mask=mk)
tf, kf = t(lambda: ub.varlen_fmha_fwd(qd, cu, 512, p_dropout=p, out=o, lse=lse, dropout_mask=mk), 0)
# the backward with the host LPT schedule of its work items (as the bench step runs it; SCHED=0: the
# kernels' snake deal)
sb = None
if os.environ.get("SCHED", "1") == "1":
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    sb = torch.from_numpy(_api.fmha_schedule(L, 16, 512, sms, True)).cuda()
tb, kb = t(lambda: ub.varlen_fmha_bwd(qd, o, lse, gd, cu, 512, p_dropout=p, dropout_mask=mk, schedule=sb), 1)
print(f"{dist} p={p} T={T} fwd call {tf:.1f} us kernel {kf:.1f} us ({4*16*64*s2/kf/1e6:.0f} TFLOP/s) | "
      f"bwd call {tb:.1f} us kernel {kb:.1f} us ({8*16*64*s2/kb/1e6:.0f} TFLOP/s strict) | "
      f"fwd+bwd calls {T/(tf+tb):.1f} Mtok/s")
