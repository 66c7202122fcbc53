"""iALS++ training entry points (host mirror of the reference ``solvers.py``).

Same names, signatures, argument meaning and errors as the reference
(``BlockPartition`` :49-64, ``EpochReport`` :67-80, ``partition_dims`` :83-92,
``block_update`` :236-252, ``ialspp_epoch`` :340-375, ``iterate_epochs``
:378-402, ``train`` :405-413).  The numerical work runs on the B200 through
``libials_b200.so``; the host only moves the factors in and out:

* ``block_update`` / ``ialspp_epoch`` take the caller's float64 NumPy model and
  cache, run on the device in FP32 and write the result back in place;
* ``train`` / ``iterate_epochs`` upload once, keep W, H and the cache resident
  for all epochs and write back before every yield (``iterate_epochs``) or
  once at the end (``train``).

``solver="ials"`` and ``solver="icd"`` run the same device sweep with b = d and
b = 1 -- the reference's own equivalence tests (``tests/test_solvers.py:125-149``)
pin those cases to its dedicated solvers.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .linalg import SingularMatrixError, check_block
from .model import FactorModel, PredictionCache, SolverConfig

__all__ = ["BlockPartition", "EpochReport", "partition_dims", "block_update", "ialspp_epoch",
           "iterate_epochs", "train", "DeviceTrainer"]


@dataclass(frozen=True)
class BlockPartition:
    """Ordered, disjoint index blocks covering every embedding dimension."""

    blocks: tuple
    dim: int

    def __post_init__(self):
        covered = np.zeros(self.dim, dtype=bool)
        for blk in self.blocks:
            blk = check_block(blk, self.dim)
            if np.any(covered[blk]):
                raise ValueError("blocks must be disjoint")
            covered[blk] = True
        if not np.all(covered):
            raise ValueError("blocks must cover every dimension")


@dataclass
class EpochReport:
    """Per-phase device seconds of one epoch (CUDA events); ``loss`` on request."""

    epoch: int
    user_seconds: float = 0.0
    item_seconds: float = 0.0
    gramian_seconds: float = 0.0
    cache_seconds: float = 0.0
    loss: float | None = None

    @property
    def train_seconds(self) -> float:
        return self.user_seconds + self.item_seconds + self.gramian_seconds + self.cache_seconds


def partition_dims(dim: int, block_size: int) -> BlockPartition:
    """Contiguous ascending blocks of ``block_size``; the last keeps the remainder."""
    dim, block_size = int(dim), int(block_size)
    if dim < 1:
        raise ValueError("dim must be positive")
    if not 1 <= block_size <= dim:
        raise ValueError("block_size must be in [1, dim]")
    return BlockPartition(tuple(np.arange(s, min(s + block_size, dim))
                                for s in range(0, dim, block_size)), dim)


def _layout(partition: BlockPartition):
    """Column permutation making the blocks contiguous, plus (b0, b) per block."""
    perm = np.concatenate([np.asarray(b, dtype=np.int64) for b in partition.blocks])
    spans, b0 = [], 0
    for blk in partition.blocks:
        spans.append((b0, len(blk)))
        b0 += len(blk)
    identity = bool(np.array_equal(perm, np.arange(partition.dim)))
    return perm, spans, identity


def _uniform_spans(spans, dim: int) -> bool:
    """True when the spans are exactly partition_dims(dim, b)'s blocks -- every
    span (b0, min(b, dim - b0)) for b0 = 0, b, 2b, ... -- which is what one
    ials_epoch call sweeps.  A wider (or narrower) last block is not."""
    b = spans[0][1]
    return list(spans) == [(s, min(b, dim - s)) for s in range(0, dim, b)]


class DeviceTrainer:
    """W, H and the cache resident on one device for a dataset + config."""

    def __init__(self, model: FactorModel, data, config: SolverConfig, partition=None,
                 device=None, cache: PredictionCache | None = None):
        import torch

        from ._runtime import default_engine_session, to_device_f32

        self.rt = default_engine_session(device)
        self.eng = self.rt.engine_for(data)
        self.eng.p.set_regularizer(config.unobserved_weight, config.reg, config.reg_exponent)
        self.config, self.model, self.data = config, model, data
        part = partition if partition is not None else partition_dims(model.dim, config.block_size)
        if part.dim != model.dim:
            raise ValueError("partition does not match the model dimension")
        self.perm, self.spans, self.identity = _layout(part)
        w, h = model.user_factors, model.item_factors
        if not self.identity:
            w, h = w[:, self.perm], h[:, self.perm]
        self.W = to_device_f32(w, self.rt.device)
        self.H = to_device_f32(h, self.rt.device)
        self.cache = torch.zeros(data.n_interactions, dtype=torch.float32, device=self.rt.device)
        if cache is not None:
            self.cache.copy_(torch.from_numpy(np.asarray(cache.scores, dtype=np.float32)))
        bmax = max(b for _, b in self.spans)
        self.slab = torch.empty((model.dim, bmax), dtype=torch.float32, device=self.rt.device)
        self.uniform = self.identity and _uniform_spans(self.spans, model.dim)

    # ---------------------------------------------------------------- passes
    def pass_(self, side, b0, b):
        e = self.eng
        slab = self.slab.view(-1)[: self.model.dim * b].view(self.model.dim, b)
        if side == "user":
            e.partial_gramian(self.H, b0, b, slab)
            e.side_pass("user", self.H, self.W, b0, b, slab, self.config.unobserved_weight,
                        self.cache)
        else:
            e.partial_gramian(self.W, b0, b, slab)
            e.side_pass("item", self.W, self.H, b0, b, slab, self.config.unobserved_weight,
                        self.cache)

    def epoch(self, index=0, timed=True) -> EpochReport:
        import torch

        rep = EpochReport(index)
        e = self.eng
        a0 = self.config.unobserved_weight
        self.rt.session.reset_singular()
        if not timed:
            if self.uniform:
                e.epoch(self.W, self.H, self.cache, self.spans[0][1], a0)
            else:
                e.predictions(self.W, self.H, self.cache)
                for b0, b in self.spans:
                    self.pass_("user", b0, b)
                    self.pass_("item", b0, b)
            self._check()
            return rep
        ev = lambda: torch.cuda.Event(enable_timing=True)
        marks = [ev()]
        marks[0].record()
        if self.uniform:
            # one ials_epoch call (tensor-core GEMMs when b in 33..128), with
            # the phase events recorded inside it
            nb = len(self.spans)
            evs = [ev() for _ in range(2 + 4 * nb)]
            e.epoch(self.W, self.H, self.cache, self.spans[0][1], a0, events=evs)
            names = ["cache"] + [n for _ in range(nb) for n in ("gramian", "user", "gramian", "item")]
            phases = list(zip(names, evs[1:]))
            prev = evs[0]
            torch.cuda.synchronize(self.rt.device)
            for name, m in phases:
                secs = prev.elapsed_time(m) / 1e3
                setattr(rep, f"{name}_seconds", getattr(rep, f"{name}_seconds") + secs)
                prev = m
            self._check()
            return rep
        e.predictions(self.W, self.H, self.cache)
        phases = [("cache", ev())]
        phases[-1][1].record()
        d = self.model.dim
        for b0, b in self.spans:
            slab = self.slab.view(-1)[: d * b].view(d, b)
            for side, fixed, own in (("user", self.H, self.W), ("item", self.W, self.H)):
                e.partial_gramian(fixed, b0, b, slab)
                phases.append(("gramian", ev()))
                phases[-1][1].record()
                e.side_pass(side, fixed, own, b0, b, slab, a0, self.cache)
                phases.append((side, ev()))
                phases[-1][1].record()
        torch.cuda.synchronize(self.rt.device)
        prev = marks[0]
        for name, m in phases:
            secs = prev.elapsed_time(m) / 1e3
            setattr(rep, f"{name}_seconds", getattr(rep, f"{name}_seconds") + secs)
            prev = m
        self._check()
        return rep

    def block(self, b0, b, side):
        self.rt.session.reset_singular()
        self.pass_(side, b0, b)
        self._check()

    def _check(self):
        from .engine import SingularBlock

        try:
            self.rt.session.raise_if_singular()
        except SingularBlock as err:
            raise SingularMatrixError(
                f"normal equations singular for row {err.row} (pivot {err.pivot})",
                pivot=err.pivot, row=err.row) from None

    def loss(self) -> float:
        return self.eng.loss(self.W, self.H, self.config.unobserved_weight)

    # ---------------------------------------------------------------- I/O
    def write_back(self, cache: PredictionCache | None = None):
        w = self.W.double().cpu().numpy()
        h = self.H.double().cpu().numpy()
        if not self.identity:
            inv = np.empty_like(self.perm)
            inv[self.perm] = np.arange(self.perm.size)
            w, h = w[:, inv], h[:, inv]
        self.model.user_factors[:] = w
        self.model.item_factors[:] = h
        if cache is not None:
            cache.scores[:] = self.cache.double().cpu().numpy()


def _check_shapes(model, data, config):
    if model.dim != config.dim:
        raise ValueError("model dimension does not match the configuration")
    if model.user_factors.shape[0] != data.num_users or \
            model.item_factors.shape[0] != data.num_items:
        raise ValueError("model shape does not match the dataset")


def block_update(model: FactorModel, data, cache: PredictionCache, config: SolverConfig,
                 block, side="user", device=None):
    """One Newton block pass over one side, maintaining the score cache."""
    block = check_block(block, model.dim)
    if side not in ("user", "item"):
        raise ValueError("side must be 'user' or 'item'")
    rest = np.setdiff1d(np.arange(model.dim), block)
    part = BlockPartition((block,) + ((rest,) if rest.size else ()), model.dim)
    tr = DeviceTrainer(model, data, config, part, device, cache)
    tr.block(0, int(block.size), side)
    tr.write_back(cache)


class _HostEpochRunner:
    """Device buffers for the float64 drop-in epoch of one dataset at one
    width on one device (cached across calls): fp32 W / H / cache, the f64
    staging of ials_epoch_host64, the row schedules and the workspace of the
    dataset's engine."""

    def __init__(self, data, dim, device):
        import torch

        from ._runtime import default_engine_session

        self.rt = default_engine_session(device)
        self.eng = self.rt.engine_for(data)
        dev = self.rt.device
        U, I, S = data.num_users, data.num_items, data.n_interactions
        self.W = torch.empty((U, dim), dtype=torch.float32, device=dev)
        self.H = torch.empty((I, dim), dtype=torch.float32, device=dev)
        self.cache = torch.empty(max(S, 1), dtype=torch.float32, device=dev)[:S]
        nbytes = int(self.eng.lib.ials_host64_staging_bytes(U, I, dim, S))
        self.staging = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)

    def epoch(self, model, cache, config, b, index):
        import torch

        from ._runtime import pin_host_array

        e = self.eng
        e.p.set_regularizer(config.unobserved_weight, config.reg, config.reg_exponent)
        for a in (model.user_factors, model.item_factors, cache.scores):
            pin_host_array(a)
        nb = -(-model.dim // b)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 + 4 * nb)]
        self.rt.session.reset_singular()
        e.epoch_host64(model.user_factors, model.item_factors, self.W, self.H, self.cache, b,
                       config.unobserved_weight, self.staging, cache_out=cache.scores, events=ev)
        torch.cuda.current_stream(self.rt.device).synchronize()
        rep = EpochReport(index)
        names = ["cache"] + [n for _ in range(nb) for n in ("gramian", "user", "gramian", "item")]
        prev = ev[0]
        for name, m in zip(names, ev[1:]):
            setattr(rep, f"{name}_seconds", getattr(rep, f"{name}_seconds") + prev.elapsed_time(m) / 1e3)
            prev = m
        return rep


_RUNNERS = None


def _host_runner(data, dim, device):
    global _RUNNERS
    import weakref

    import torch
    if _RUNNERS is None:
        _RUNNERS = weakref.WeakKeyDictionary()
    idx = torch.cuda.current_device() if device is None else (torch.device(device).index or 0)
    try:
        per = _RUNNERS.setdefault(data, {})
    except TypeError:
        per = {}
    run = per.get((dim, idx))
    if run is None:
        run = per[(dim, idx)] = _HostEpochRunner(data, dim, device)
    return run


def _f64_c(a) -> bool:
    return isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous and \
        a.flags.writeable


def ialspp_epoch(model: FactorModel, data, cache: PredictionCache, config: SolverConfig,
                 partition: BlockPartition | None = None, epoch_index: int = 0,
                 device=None) -> EpochReport:
    """Block epoch: recompute the cache, then per block a user and an item pass.

    The caller's float64 model and cache are updated in place.  With the
    default contiguous partition (or ``partition_dims``' own blocks) the epoch
    is one ``ials_epoch_host64`` call: the f64 arrays are page-locked in place
    once and copied through device staging with the casts on the GPU,
    overlapped with the epoch, and the device buffers are kept across calls
    for the same dataset.  Other partitions permute columns on the host."""
    part = partition if partition is not None else partition_dims(model.dim, config.block_size)
    if part.dim != model.dim:
        raise ValueError("partition does not match the model dimension")
    from .model import _check_pair
    _check_pair(model, data)                 # compute_predictions' checks (model.py:153-165)
    if cache.scores.shape != (data.n_interactions,):
        raise ValueError("cache length does not match the dataset")
    perm, spans, identity = _layout(part)
    if (identity and _uniform_spans(spans, model.dim) and data.n_interactions > 0
            and all(_f64_c(a) for a in (model.user_factors, model.item_factors, cache.scores))):
        return _host_runner(data, model.dim, device).epoch(model, cache, config, spans[0][1],
                                                           epoch_index)
    tr = DeviceTrainer(model, data, config, partition, device, cache)
    rep = tr.epoch(epoch_index)
    tr.write_back(cache)
    return rep


def ials_epoch(model: FactorModel, data, config: SolverConfig, epoch_index: int = 0,
               device=None) -> EpochReport:
    """Full-vector epoch (solvers.py:275-300): an exact user pass, then an
    exact item pass.  On the device this is the block sweep with one block of
    width d: a Newton step from an exact cache solves the row's quadratic in
    closed form, so it equals the reference's direct solve (pinned by the
    reference's own equivalence test, test_solvers.py:125-149).  Widths
    above 256 take the batched wide solver (csrc/ials_sweep_wide.cuh).  The
    cache is internal and discarded, as in the reference."""
    cache = PredictionCache(np.zeros(data.n_interactions))
    return ialspp_epoch(model, data, cache, config, partition_dims(model.dim, model.dim),
                        epoch_index, device)


def icd_epoch(model: FactorModel, data, cache: PredictionCache, config: SolverConfig,
              epoch_index: int = 0, device=None) -> EpochReport:
    """Coordinate epoch (solvers.py:303-337): per dimension a user and an item
    pass with the cache maintained; the block sweep with width 1."""
    return ialspp_epoch(model, data, cache, config, partition_dims(model.dim, 1), epoch_index,
                        device)


def coordinate_update(model: FactorModel, data, cache: PredictionCache, config: SolverConfig,
                      dim_index: int, side="user", device=None):
    """One scalar-coordinate pass over one side (solvers.py:255-272)."""
    f = int(dim_index)
    if not 0 <= f < model.dim:
        raise ValueError("dim_index out of range")
    if side not in ("user", "item"):
        raise ValueError("side must be 'user' or 'item'")
    block_update(model, data, cache, config, np.array([f]), side, device)


def _solver_partition(config: SolverConfig):
    if config.solver == "ials":
        return partition_dims(config.dim, config.dim)
    if config.solver == "icd":
        return partition_dims(config.dim, 1)
    return partition_dims(config.dim, config.block_size)


def iterate_epochs(model: FactorModel, data, config: SolverConfig, log_loss: bool = False,
                   device=None):
    """Train in place, yielding one :class:`EpochReport` per epoch."""
    _check_shapes(model, data, config)
    if config.epochs == 0:
        return
    tr = DeviceTrainer(model, data, config, _solver_partition(config), device)
    for epoch in range(config.epochs):
        rep = tr.epoch(epoch)
        if log_loss:
            rep.loss = tr.loss()
        tr.write_back()
        yield rep


def train(model: FactorModel, data, config: SolverConfig, log_loss: bool = False, device=None):
    """Run ``config.epochs`` epochs; returns ``(model, reports)`` (in place)."""
    _check_shapes(model, data, config)
    reports = []
    if config.epochs == 0:
        return model, reports
    tr = DeviceTrainer(model, data, config, _solver_partition(config), device)
    for epoch in range(config.epochs):
        rep = tr.epoch(epoch)
        if log_loss:
            rep.loss = tr.loss()
        reports.append(rep)
    tr.write_back()
    return model, reports
