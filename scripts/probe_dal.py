"""Dev probe: DAL fwd/bwd kernel time (library events) at p = 0 and 0.1, E = 1024, T = 15157."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2208_08124_b200 as ub
from paper_2208_08124_b200 import api
T, E = 15157, 1024
hs = [tuple(torch.randn((T, E), device="cuda").to(torch.bfloat16) for _ in range(3)) for _ in range(3)]
g = torch.ones(E, dtype=torch.bfloat16, device="cuda"); b = torch.zeros(E, dtype=torch.bfloat16, device="cuda")
for p in (0.0, 0.1):
    st = [ub.dal_fwd(h[0], h[1], g, b, p, 1e-12, 5) for h in hs]
    for name, kid, fn, nb in (("fwd", api.PROF_DAL_FWD, lambda k: ub.dal_fwd(hs[k][0], hs[k][1], g, b, p, 1e-12, 5), 6 * T * E),
                              ("bwd", api.PROF_DAL_BWD, lambda k: ub.dal_bwd(hs[k][2], hs[k][0], hs[k][1], g, st[k][1], st[k][2], p, 5), 10 * T * E)):
        for k in range(3): fn(k)
        torch.cuda.synchronize(); torch.cuda._sleep(2_000_000)
        ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(20)]
        for k in range(20):
            api.profile_events(kid, *ev[k]); fn(k % 3)
        api.profile_events(kid); torch.cuda.synchronize()
        us = float(np.median([a.elapsed_time(c) for a, c in ev])) * 1e3
        print(f"p={p} {name}: {us:.1f} us  {nb / us / 1e3:.0f} GB/s")
