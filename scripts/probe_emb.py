"""Dev probe: embedding bwd time vs id distribution (uniform vs Zipf)."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2208_08124_b200 as ub
T, E, V = 15157, 1024, 30522
rng = np.random.default_rng(0)
pos = torch.from_numpy((np.arange(T) % 512).astype(np.int32)).cuda()
seg = torch.from_numpy((rng.random(T) < 0.5).astype(np.int32)).cuda()
dout = torch.randn((T, E), device="cuda").to(torch.bfloat16)
for name, ids_np in (("uniform", rng.integers(0, V, T)), ("zipf1.1", np.minimum(rng.zipf(1.1, T) - 1, V - 1)),
                     ("zipf1.2", np.minimum(rng.zipf(1.2, T) - 1, V - 1))):
    ids = torch.from_numpy(ids_np.astype(np.int32)).cuda()
    dws = [torch.zeros((n, E), dtype=torch.float32, device="cuda") for n in (V, 512, 2)]
    for _ in range(2): ub.embedding_bwd(dout, ids, pos, seg, *dws)
    torch.cuda.synchronize(); torch.cuda._sleep(2_000_000)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): ub.embedding_bwd(dout, ids, pos, seg, *dws)
    e1.record(); torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us, top-id share {np.bincount(ids_np).max() / T:.3f}")
# context: PyTorch's embedding backward (sort-based) on the same ids, fp32 weights
for name, ids_np in (("uniform", rng.integers(0, V, T)), ("zipf1.2", np.minimum(rng.zipf(1.2, T) - 1, V - 1))):
    ids = torch.from_numpy(ids_np.astype(np.int64)).cuda()
    w = torch.zeros((V, E), dtype=torch.float32, device="cuda", requires_grad=True)
    g = dout.float()
    def run():
        out = torch.nn.functional.embedding(ids, w)
        out.backward(g)
    for _ in range(2): run()
    torch.cuda.synchronize(); torch.cuda._sleep(2_000_000)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): run()
    e1.record(); torch.cuda.synchronize()
    print(f"torch {name}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us (word table only, incl. its forward)")
