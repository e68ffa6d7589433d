"""Dev probe: gather kernels vs torch copy / fill bandwidth on the config-2 hidden state."""
import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2208_08124_b200 as ub
from paper_2208_08124_b200 import api
import synth
L = synth.gen_lengths("mlperf_like_v0", 56, 0)
off = np.concatenate([[0], np.cumsum(L)]).astype(np.int32)
T = int(off[-1]); B, S, E = 56, 512, 1024
cu = torch.tensor(off).cuda()
sets = [(torch.randn(B, S, E, device="cuda").bfloat16(), torch.empty(T, E, device="cuda", dtype=torch.bfloat16),
         torch.empty(T, E, device="cuda", dtype=torch.bfloat16)) for _ in range(3)]
import os
NITER = int(os.environ.get("PROBE_N", "30"))
def t(fn, n=NITER):
    for k in range(3): fn(sets[k])
    torch.cuda.synchronize(); torch.cuda._sleep(2_000_000)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for k in range(n): fn(sets[k % 3])
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
row = E * 2
for name, fn, nb in (("torch copy packed", lambda s: s[2].copy_(s[1]), 2 * T * row),
                     ("torch zero padded", lambda s: s[0].zero_(), B * S * row),
                     ("ub unpad", lambda s: ub.unpad(s[0], cu, T, out=s[1]), 2 * T * row),
                     ("ub pad", lambda s: ub.pad(s[1], cu, B, S, out=s[0]), T * row + B * S * row)):
    us = t(fn)
    print(f"{name:20s} {us:7.2f} us  {nb / us / 1e3:7.0f} GB/s")
# a5 reorder (exchange copy) at the stress record size (a bf16 hidden row per token), one rank
rec = E * 2
perm = api.balance_plan(L, 1, B, S, "paper")["perm"]
d_unpack = torch.from_numpy(api.exchange_tables(L, perm, 1, B, 0, unpack=True)[0]).cuda()
xs = [(torch.randint(0, 255, (T, rec), dtype=torch.uint8, device="cuda"), torch.empty((T, rec), dtype=torch.uint8,
       device="cuda")) for _ in range(3)]
def t2(fn, n=NITER):
    for k in range(3): fn(xs[k])
    torch.cuda.synchronize(); torch.cuda._sleep(2_000_000)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for k in range(n): fn(xs[k % 3])
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
us = t2(lambda x: api.exchange_copy(x[0], x[1], None, None, d_unpack, B, rec, 0))
print(f"{'ub exchange_copy':20s} {us:7.2f} us  {2 * T * rec / us / 1e3:7.0f} GB/s")
