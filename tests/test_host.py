"""CPU-only tests of the host mirror: CSR construction (bit-exact vs the
reference goldens), validation errors, configuration, partitions, init,
the row scheduler and the synthetic generator."""

import numpy as np
import pytest

from conftest import small_case

import paper_2110_14044_b200 as ials
from paper_2110_14044_b200 import synthetic
from paper_2110_14044_b200.engine import plan_schedule


def test_csr_bit_exact_tiny(tiny_golden):
    g = tiny_golden
    data = ials.InteractionDataset(int(g["num_users"]), int(g["num_items"]), g["coo_users"],
                                   g["coo_items"])
    assert np.array_equal(data.users, g["csr_users"])
    assert np.array_equal(data.items, g["csr_items"])
    assert np.array_equal(data.user_ptr, g["user_ptr"])
    assert np.array_equal(data.item_ptr, g["item_ptr"])
    assert np.array_equal(data.item_view().cache_pos, g["item_order"])
    iv = data.item_view()
    assert np.array_equal(iv.cols, data.users[data.item_order])
    # both views hold the same multiset of (user, item) pairs
    uv = data.user_view()
    a = np.sort(np.repeat(np.arange(data.num_users), uv.counts) * data.num_items + uv.cols)
    b = np.sort(iv.cols * data.num_items + np.repeat(np.arange(data.num_items), iv.counts))
    assert np.array_equal(a, b)


@pytest.mark.parametrize("seed", list(range(1, 11)))
def test_csr_bit_exact_small(small_golden, seed):
    c = small_case(small_golden, seed)
    data = ials.InteractionDataset(c["U"], c["I"], c["users"], c["items"], c["labels"], c["weights"])
    assert np.array_equal(data.user_ptr, c["user_ptr"])
    assert np.array_equal(data.item_ptr, c["item_ptr"])
    assert np.array_equal(data.item_view().cache_pos, c["item_order"])
    assert np.array_equal(data.items, c["csr_items"])


def test_synthetic_digest_and_shape():
    U, I, u, i = synthetic.generate("tiny", 0)
    assert (U, I, u.size) == (2000, 1000, 50000)
    assert synthetic.digest(u, i).startswith("a9c031a5f7dac8e1")
    counts = np.bincount(u, minlength=U)
    assert counts.min() >= 1 and 18 <= np.median(counts) <= 22
    pairs = u * I + i
    assert np.unique(pairs).size == pairs.size           # sampled without replacement
    again = synthetic.generate("tiny", 0)
    assert np.array_equal(again[2], u) and np.array_equal(again[3], i)


@pytest.mark.parametrize("kwargs", [
    dict(users=[0, 1], items=[0]),            # length mismatch
    dict(users=[0, 5], items=[0, 1]),         # user out of range
    dict(users=[0, 1], items=[0, 9]),         # item out of range
    dict(users=[0, 1], items=[0, 1], labels=[1.0, np.nan]),
    dict(users=[0, 1], items=[0, 1], weights=[1.0, 0.0]),
])
def test_dataset_validation(kwargs):
    with pytest.raises(ValueError):
        ials.InteractionDataset(3, 3, **kwargs)
    with pytest.raises(ValueError):
        ials.InteractionDataset(0, 3, [], [])


def test_empty_dataset_and_duplicates():
    data = ials.InteractionDataset(3, 2, [2, 0, 2, 2], [1, 0, 1, 0])
    assert data.n_interactions == 4
    assert list(data.user_counts) == [1, 0, 3] and list(data.item_counts) == [2, 2]
    assert list(data.items) == [0, 1, 1, 0]           # stable within user 2
    empty = ials.InteractionDataset(2, 2, [], [])
    assert empty.n_interactions == 0 and list(empty.user_ptr) == [0, 0, 0]


@pytest.mark.parametrize("kw", [dict(dim=0), dict(dim=4, block_size=5), dict(dim=4, reg=0.0),
                                dict(dim=4, unobserved_weight=-1), dict(dim=4, solver="x"),
                                dict(dim=4, epochs=-1), dict(dim=4, init_stddev=0),
                                dict(dim=4, threads=-1), dict(dim=4, reg_exponent=-1)])
def test_config_validation(kw):
    with pytest.raises(ValueError):
        ials.SolverConfig(**kw)


def test_config_defaults():
    c = ials.SolverConfig(dim=200)
    assert c.block_size == 64 and c.solver == "ialspp"
    assert ials.SolverConfig(dim=10).block_size == 10


def test_partition_rules():
    assert [b.tolist() for b in ials.partition_dims(10, 4).blocks] == [[0, 1, 2, 3], [4, 5, 6, 7], [8, 9]]
    assert [b.tolist() for b in ials.partition_dims(5, 5).blocks] == [[0, 1, 2, 3, 4]]
    for bad in (0, 6, -1):
        with pytest.raises(ValueError):
            ials.partition_dims(5, bad)
    with pytest.raises(ValueError):
        ials.BlockPartition((np.array([0, 1]), np.array([1, 2])), 3)     # overlap
    with pytest.raises(ValueError):
        ials.BlockPartition((np.array([0, 1]),), 3)                      # not covering
    with pytest.raises(ValueError):
        ials.BlockPartition((np.array([1, 0]), np.array([2])), 3)        # not increasing


def test_check_block():
    assert list(ials.check_block([0, 2], 3)) == [0, 2]
    for bad in ([], [3], [-1], [1, 1], [2, 1]):
        with pytest.raises(ValueError):
            ials.check_block(bad, 3)


def test_init_model_matches_reference(tiny_golden):
    cfg = ials.SolverConfig(dim=32, block_size=8, seed=0, init_stddev=0.1)
    m = ials.init_model(cfg, 2000, 1000)
    assert np.array_equal(m.user_factors.astype(np.float32), tiny_golden["w0"])
    assert np.array_equal(m.item_factors.astype(np.float32), tiny_golden["h0"])


def test_effective_reg():
    cfg = ials.SolverConfig(dim=2, unobserved_weight=0.5, reg=0.1, reg_exponent=1.0)
    assert np.allclose(ials.effective_reg(np.array([0, 4]), 10, cfg), [0.5, 0.9])
    cfg0 = cfg.with_(reg_exponent=0.0)
    assert np.allclose(ials.effective_reg(np.array([0, 4]), 10, cfg0), [0.1, 0.1])


@pytest.mark.parametrize("thr,sl", [(4, 2), (5, 3), (100, 10)])
def test_plan_schedule_covers_every_entry_once(thr, sl):
    rng = np.random.default_rng(3)
    counts = np.concatenate([rng.integers(0, 12, 40), [0, 0, 31, 9]])
    ptr = np.concatenate([[0], np.cumsum(counts)])
    plan = plan_schedule(ptr, thr, sl)
    rows = np.concatenate([plan["light"], plan["heavy"]])
    assert np.array_equal(np.sort(rows), np.arange(counts.size))
    assert np.all(counts[plan["light"]] <= thr) and np.all(counts[plan["heavy"]] > thr)
    assert np.all(np.diff(counts[plan["light"]]) <= 0)               # LPT order
    covered = np.zeros(ptr[-1], dtype=int)
    for h, (b, e) in zip(plan["slice_heavy"], zip(plan["beg"], plan["end"])):
        r = plan["heavy"][h]
        assert ptr[r] <= b < e <= ptr[r + 1] and e - b <= sl
        covered[b:e] += 1
    heavy_entries = np.concatenate([np.arange(ptr[r], ptr[r + 1]) for r in plan["heavy"]] or [[]])
    assert np.all(covered[heavy_entries.astype(int)] == 1) and covered.sum() == heavy_entries.size
    assert plan["slice0"][-1] == plan["beg"].size


def test_no_cpu_fallback_without_device(monkeypatch):
    """The solver must fail loudly without CUDA, never compute on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    data = ials.InteractionDataset(2, 2, [0, 1], [0, 1])
    cfg = ials.SolverConfig(dim=2, epochs=1)
    model = ials.init_model(cfg, 2, 2)
    with pytest.raises(RuntimeError):
        ials.train(model, data, cfg)
    with pytest.raises(RuntimeError):
        ials.compute_predictions(model, data)


def test_uniform_spans_only_for_partition_dims():
    """a contiguous partition whose last block is wider than the
    first is not partition_dims(d, b) and must not go to one ials_epoch call."""
    from paper_2110_14044_b200.solvers import _layout, _uniform_spans
    for d, b in ((30, 10), (30, 7), (8, 8), (13, 1)):
        _, spans, ident = _layout(ials.partition_dims(d, b))
        assert ident and _uniform_spans(spans, d)
    wide_last = ials.BlockPartition((np.arange(0, 10), np.arange(10, 30)), 30)
    _, spans, ident = _layout(wide_last)
    assert ident and not _uniform_spans(spans, 30)
    narrow_mid = ials.BlockPartition((np.arange(0, 10), np.arange(10, 15), np.arange(15, 30)), 30)
    assert not _uniform_spans(_layout(narrow_mid)[1], 30)
