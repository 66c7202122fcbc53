"""Device CSR construction (ials_build_csr) is bit-exact
with the reference's host build (InteractionDataset.__init__ / user_view /
item_view, data.py:98-134,148-162): against the reference-generated goldens,
and against the host mirror (itself pinned to those goldens) on ragged,
duplicated, empty-row, single-key and full-size shapes."""

import numpy as np
import pytest

from conftest import small_case

import paper_2110_14044_b200 as ials

pytestmark = pytest.mark.gpu


def _check(U, I, users, items):
    from paper_2110_14044_b200.csr import build_csr_device
    ref = ials.InteractionDataset(U, I, users, items)
    got = build_csr_device(U, I, users, items)
    g = lambda t: t.cpu().numpy().astype(np.int64)
    order = np.argsort(np.asarray(users, dtype=np.int64), kind="stable")
    assert np.array_equal(g(got.order), order)
    assert np.array_equal(g(got.user_ptr), ref.user_ptr)
    assert np.array_equal(g(got.user_cols), ref.items)
    assert np.array_equal(g(got.item_ptr), ref.item_ptr)
    iv = ref.item_view()
    assert np.array_equal(g(got.item_pos), iv.cache_pos)
    assert np.array_equal(g(got.item_cols), iv.cols)
    return got


def test_tiny_golden(tiny_golden):
    g = tiny_golden
    from paper_2110_14044_b200.csr import build_csr_device
    got = build_csr_device(int(g["num_users"]), int(g["num_items"]), g["coo_users"], g["coo_items"])
    assert np.array_equal(got.user_ptr.cpu().numpy(), g["user_ptr"])
    assert np.array_equal(got.item_ptr.cpu().numpy(), g["item_ptr"])
    assert np.array_equal(got.user_cols.cpu().numpy(), g["csr_items"])
    assert np.array_equal(got.item_pos.cpu().numpy(), g["item_order"])
    assert np.array_equal(got.item_cols.cpu().numpy(), g["csr_users"][g["item_order"]])


@pytest.mark.parametrize("seed", list(range(1, 11)))
def test_small_goldens(small_golden, seed):
    c = small_case(small_golden, seed)
    got = _check(c["U"], c["I"], c["users"], c["items"])
    assert np.array_equal(got.user_ptr.cpu().numpy(), c["user_ptr"])
    assert np.array_equal(got.item_pos.cpu().numpy(), c["item_order"])


@pytest.mark.parametrize("U,I,n,seed", [
    (1, 1, 17, 0),            # one key: zero radix passes
    (300, 1, 5000, 1),        # one item
    (256, 257, 9000, 2),      # one / two passes at the digit boundary
    (5000, 3000, 0, 3),       # no interactions
    (70000, 300, 40000, 4),   # most users empty, runs of empty rows
    (136677, 20108, 600000, 5),   # ML20M-shaped id ranges (3 + 2 passes)
    (571355, 41140, 300000, 6),   # MSD-shaped id ranges
    (3, 2 ** 24 + 5, 50000, 7),   # item ids above 2^24: four passes
])
def test_random_shapes(U, I, n, seed):
    rng = np.random.default_rng(seed)
    users = rng.integers(0, U, n)
    items = np.minimum(rng.zipf(1.2, n) - 1, I - 1) if I > 1 else np.zeros(n, dtype=np.int64)
    users[: n // 3] = users[n // 3: 2 * (n // 3)]   # duplicated (user, item) pairs stay distinct
    items[: n // 3] = items[n // 3: 2 * (n // 3)]
    _check(U, I, users, items)


def test_validation_matches_reference():
    from paper_2110_14044_b200.csr import build_csr_device
    with pytest.raises(ValueError, match="user index out of range"):
        build_csr_device(3, 3, [0, 3], [0, 1])
    with pytest.raises(ValueError, match="item index out of range"):
        build_csr_device(3, 3, [0, 1], [0, -1])
    with pytest.raises(ValueError, match="equal length"):
        build_csr_device(3, 3, [0, 1], [0])
    with pytest.raises(ValueError, match="at least one user"):
        build_csr_device(0, 3, [], [])


def test_full_size_synthetic_properties():
    """configs[1] shape (10.0M pairs): both views are permutations of the same
    multiset, rows sorted stably (canonical positions increase inside every
    item row), and the pointers match the host bincount."""
    from paper_2110_14044_b200 import synthetic
    from paper_2110_14044_b200.csr import build_csr_device
    U, I, users, items = synthetic.generate("mid", 0)
    got = build_csr_device(U, I, users, items)
    up = got.user_ptr.cpu().numpy()
    ip = got.item_ptr.cpu().numpy()
    assert np.array_equal(np.diff(up), np.bincount(users, minlength=U))
    assert np.array_equal(np.diff(ip), np.bincount(items, minlength=I))
    order = got.order.cpu().numpy()
    assert np.array_equal(order, np.argsort(users, kind="stable"))
    pos = got.item_pos.cpu().numpy()
    assert np.array_equal(np.sort(pos), np.arange(users.size))
    # stable: inside each item row the canonical positions increase
    d = np.diff(pos)
    starts = ip[1:-1]
    mask = np.ones(d.size, dtype=bool)
    mask[starts[(starts > 0) & (starts < users.size)] - 1] = False
    assert (d[mask] > 0).all()
    assert np.array_equal(got.item_cols.cpu().numpy(), users[order][pos])


def test_device_csr_drives_an_epoch():
    """An epoch on the device-built CSR equals the epoch on the host-built one
    bit for bit (same arrays, same schedule, deterministic kernels)."""
    import torch
    from paper_2110_14044_b200.csr import build_csr_device
    from paper_2110_14044_b200.engine import DeviceProblem, Engine
    rng = np.random.default_rng(9)
    U, I, n, d, b = 900, 300, 20000, 128, 128
    users = rng.integers(0, U, n)
    items = np.minimum(rng.zipf(1.2, n) - 1, I - 1)
    dev = torch.device("cuda", 0)
    out = []
    for prob in (DeviceProblem.from_dataset(ials.InteractionDataset(U, I, users, items), dev),
                 DeviceProblem.from_device_csr(build_csr_device(U, I, users, items))):
        prob.set_regularizer(0.1, 1e-3, 1.0)
        eng = Engine(prob)
        g = torch.Generator(device=dev).manual_seed(0)
        W = torch.randn(U, d, device=dev, generator=g) * 0.01
        H = torch.randn(I, d, device=dev, generator=g) * 0.01
        cache = torch.zeros(n, device=dev)
        eng.epoch(W, H, cache, b, 0.1)
        out.append((W.cpu(), H.cpu(), cache.cpu()))
    for a, c in zip(out[0], out[1]):
        assert torch.equal(a, c)
