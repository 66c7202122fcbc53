import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2110_14044_b200 as ials
from paper_2110_14044_b200 import _lib
from test_gpu_parity import _heavy_instance
lib = _lib.load()
d, b = int(sys.argv[1]), int(sys.argv[2])
U, I, users, items = _heavy_instance(3000, 900, 60, 1.0, 5)
data = ials.InteractionDataset(U, I, users, items)
cfg = ials.SolverConfig(dim=d, block_size=b, unobserved_weight=0.1, reg=1e-3, reg_exponent=1.0, epochs=1, seed=2)
init = ials.init_model(cfg, U, I)
res = {}
for tc in (0, 1):
    lib.ials_set_tensor_cores(tc)
    m = init.copy()
    cache = ials.compute_predictions(m, data)
    try:
        ials.block_update(m, data, cache, cfg, np.arange(b0 := 0, b), side="user")
    except Exception as e:
        print("tc", tc, "user err", e)
    res[tc] = m.user_factors.copy()
    print("tc", tc, "nan", np.isnan(m.user_factors).sum(), "W[0,:4]", m.user_factors[0, :4])
print("user block diff", np.abs(res[0] - res[1]).max())
for tc in (0, 1):
    lib.ials_set_tensor_cores(tc)
    m = init.copy()
    cache = ials.compute_predictions(m, data)
    try:
        ials.block_update(m, data, cache, cfg, np.arange(b), side="item")
    except Exception as e:
        print("tc", tc, "item err", e)
    res[tc] = m.item_factors.copy()
    print("item tc", tc, "nan rows", np.isnan(m.item_factors).any(1).sum(), "cache nan", np.isnan(cache.scores).sum())
print("item block diff", np.abs(res[0] - res[1]).max())
lib.ials_set_tensor_cores(1)
m = init.copy()
cache = ials.compute_predictions(m, data)
ials.block_update(m, data, cache, cfg, np.arange(b), side="item")
bad = np.where(np.isnan(m.item_factors).any(1))[0]
cnt = data.item_counts
print("nan item rows", bad.size, "of", I, "counts of bad", cnt[bad][:10], "max count", cnt.max(), "nan cols", np.where(np.isnan(m.item_factors).any(0))[0][:10])
print("cache nan", np.isnan(cache.scores).sum())
