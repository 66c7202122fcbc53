"""Check that the C-ABI epoch captures into a CUDA graph and replays to the
same result as the eager epoch; time both."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2110_14044_b200.engine import DeviceProblem, Engine
cfg = sys.argv[1] if len(sys.argv) > 1 else "tiny"
shape, d, b, _ = bench.CONFIGS[cfg]
ds = bench.dataset(shape)
U, I, S = int(ds["U"]), int(ds["I"]), int(ds["user_ptr"][-1])
dev = torch.device("cuda", 0)
prob = DeviceProblem(dev, U, I, ds["user_ptr"], ds["user_cols"], ds["item_ptr"], ds["item_cols"], ds["item_pos"])
prob.set_regularizer(0.1, 1e-3, 1.0)
eng = Engine(prob)
g = torch.Generator(device=dev).manual_seed(0)
W0 = torch.randn(U, d, device=dev, generator=g) * (0.1 / d ** 0.5)
H0 = torch.randn(I, d, device=dev, generator=g) * (0.1 / d ** 0.5)
W, H, c = W0.clone(), H0.clone(), torch.zeros(S, device=dev)
eng.epoch(W, H, c, b, 0.1); eng.epoch(W, H, c, b, 0.1)
We = W.clone()
W.copy_(W0); H.copy_(H0)
eng.epoch_graph(W, H, c, b, 0.1)          # captures (runs one eager epoch first)
W.copy_(W0); H.copy_(H0)
eng.epoch_graph(W, H, c, b, 0.1); eng.epoch_graph(W, H, c, b, 0.1)
torch.cuda.synchronize()
print("graph vs eager max |dW|:", float((W - We).abs().max()))
for name, fn in (("eager", lambda: eng.epoch(W, H, c, b, 0.1)), ("graph", lambda: eng.epoch_graph(W, H, c, b, 0.1))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): fn()
    z.record(); torch.cuda.synchronize()
    print(cfg, name, "ms/epoch", a.elapsed_time(z) / 20)
