"""Collectives: reference ring semantics on device buffers, in one process or
across processes.

Mirrors pkg/src/tenvec/comm.py:1-284 at two levels:

* In-process (every rank's buffer lives in this process, as in the
  reference): ``ring_all_reduce`` / ``ring_all_reduce_mixed`` run ONE fold
  kernel over the p device buffers (``tv_rank_fold``) that replays the
  reference's value order -- the ascending-rank sum (comm.py:95-97) or the
  mixed ring where chunk c starts at rank c and each hop computes
  demote(promote + promote) (comm.py:123-130) -- so results are bit-equal to
  the reference.  ``WorkerGroup`` keeps the threads-as-ranks rendezvous
  (comm.py:168-284) on top of them.

* One process per GPU (``RankGroup``): the same values over a transport
  (transport.py: torch.distributed + symmetric memory, or the one-GPU
  loopback of thread-ranks).  Default "fused": dtvc's split-mode contraction
  stores each owner's output range straight into that owner's peer memory,
  the owner folds with the same kernel and every rank gathers the folded
  ranges (``tvc_reduce_fused``).  "exact": an all-to-all of ring chunks in
  the storage format (reduced precision on the wire for the mixed modes),
  the fold on rank c, an all-gather -- a ring allreduce's traffic.  "p2p":
  that fold straight from the peers' buffers.  All three are bit-identical
  to the reference and across ranks; "nccl" (ncclAllReduce) is
  rank-consistent but not reference-ordered.  Device barriers over peer
  memory carry the reference's timeout semantics (CollectiveTimeout naming
  the absent ranks).

Counters follow the reference's ring accounting (comm.py:64-81).
"""

from __future__ import annotations

import collections
import contextlib
import ctypes
import os
import threading
import time
import warnings
from dataclasses import dataclass
from typing import Callable

import torch

from . import _lib
from .errors import CollectiveError, CollectiveTimeout
from .precision import PrecisionMode, tv_dtype_of
from .tensor import as_bits
from .transport import TV_PEER_HEADER, PeerBuffer, PeerMemoryUnavailable, TorchTransport

__all__ = [
    "CollectiveError", "CollectiveTimeout", "CommCounters", "ring_chunks", "ring_all_reduce",
    "ring_all_reduce_mixed", "ring_all_gather", "WorkerGroup", "RankGroup", "device_fold",
    "FusedPlan", "fused_plan", "PeerMemoryUnavailable",
]


@dataclass
class CommCounters:
    elements_sent: int = 0
    elements_received: int = 0
    touched_elements: int = 0
    collective_calls: int = 0

    def add(self, other: "CommCounters") -> None:
        self.elements_sent += other.elements_sent
        self.elements_received += other.elements_received
        self.touched_elements += other.touched_elements
        self.collective_calls += other.collective_calls


def ring_chunks(n: int, p: int) -> list[tuple[int, int]]:
    """ceil(n/p)-sized chunks with a short (possibly empty) tail (comm.py:58-61)."""
    q = -(-n // p) if n else 0
    return [(min(i * q, n), min((i + 1) * q, n)) for i in range(p)]


def ring_sizes(n: int, p: int):
    return (b - a for a, b in ring_chunks(n, p))


def _charge(counters, sender: int, receiver: int, size: int) -> None:
    if counters is None or size == 0:
        return
    counters[sender].elements_sent += size
    counters[sender].touched_elements += size
    counters[receiver].elements_received += size
    counters[receiver].touched_elements += size


def _charge_allreduce_movement(counters, sizes: list[int], p: int) -> None:
    # reduce-scatter then allgather, as the reference charges them (comm.py:73-81)
    for t in range(p - 1):
        for r in range(p):
            _charge(counters, r, (r + 1) % p, sizes[(r - t) % p])
    for t in range(p - 1):
        for r in range(p):
            _charge(counters, r, (r + 1) % p, sizes[(r + 1 - t) % p])


def _charge_allgather(counters, sizes: list[int], p: int) -> None:
    for t in range(p - 1):
        for r in range(p):
            _charge(counters, r, (r + 1) % p, sizes[(r - t) % p])


def _pair_for(buf: torch.Tensor, mode: PrecisionMode | None) -> tuple[int, int]:
    if mode is not None:
        return mode.tv_storage, mode.tv_compute
    st = tv_dtype_of(buf)
    return st, (_lib.TV_F64 if st == _lib.TV_F64 else _lib.TV_F32)


def device_fold(srcs: list[torch.Tensor], dst: torch.Tensor, *, mixed: bool,
                mode: PrecisionMode | None, chunk: int = 0, start: int = 0) -> None:
    """tv_rank_fold over p device buffers of equal length (dst may be srcs[0])."""
    p = len(srcs)
    n = dst.numel()
    st, ct = _pair_for(dst, mode)
    arr = (ctypes.c_void_p * p)(*[s.data_ptr() for s in srcs])
    lib = _lib.load()
    _lib.check(lib.tv_rank_fold(arr, p, n, chunk, start, st, ct, int(mixed), dst.data_ptr(),
                                _lib.stream_ptr()), "rank fold")


def device_fold_strided(recv: torch.Tensor, stride: int, p: int, n: int, dst: torch.Tensor, *,
                        mixed: bool, mode: PrecisionMode | None, start: int, chunk: int = 0) -> None:
    """Fold p contributions laid out back to back in one receive buffer: one
    ring chunk starting at rank `start` (chunk = 0), or whole buffers whose
    chunk c (of `chunk` elements) starts at rank c."""
    if n == 0:
        return
    st, ct = _pair_for(dst, mode)
    lib = _lib.load()
    _lib.check(lib.tv_rank_fold_strided(recv.data_ptr(), stride, p, n, chunk, start, st, ct,
                                        int(mixed), dst.data_ptr(), _lib.stream_ptr()),
               "rank fold")


SMALL_GATHER_BYTES = 1 << 20


def _check_lengths(bufs) -> int:
    n = bufs[0].numel()
    if any(b.numel() != n for b in bufs):
        raise CollectiveError("allreduce buffers differ in length across ranks")
    return n


def ring_all_reduce(bufs: list[torch.Tensor], counters: list[CommCounters] | None = None) -> None:
    """Exact-width allreduce, in place, ascending rank-order sum (comm.py:84-100)."""
    p = len(bufs)
    n = _check_lengths(bufs)
    if counters is not None:
        for c in counters:
            c.collective_calls += 1
    if p == 1:
        return
    device_fold(bufs, bufs[0], mixed=False, mode=None)
    _charge_allreduce_movement(counters, [b - a for a, b in ring_chunks(n, p)], p)
    src = as_bits(bufs[0])
    for b in bufs[1:]:
        as_bits(b).copy_(src)


def ring_all_reduce_mixed(bufs: list[torch.Tensor], mode: PrecisionMode,
                          counters: list[CommCounters] | None = None) -> None:
    """Mixed-width allreduce (comm.py:103-134): chunk c starts at rank c, every
    hop demotes.  All buffers end with identical storage bits."""
    p = len(bufs)
    n = _check_lengths(bufs)
    if counters is not None:
        for c in counters:
            c.collective_calls += 1
    if p == 1:
        return
    chunks = ring_chunks(n, p)
    device_fold(bufs, bufs[0], mixed=True, mode=mode, chunk=chunks[0][1] - chunks[0][0])
    _charge_allreduce_movement(counters, [b - a for a, b in chunks], p)
    src = as_bits(bufs[0])
    for b in bufs[1:]:
        as_bits(b).copy_(src)


def ring_all_gather(locals_: list[torch.Tensor], counters: list[CommCounters] | None = None
                    ) -> torch.Tensor:
    """Rank-order concatenation (comm.py:137-153); blocks may differ in length."""
    p = len(locals_)
    if counters is not None:
        for c in counters:
            c.collective_calls += 1
    dtype = locals_[0].dtype
    out = torch.cat([as_bits(x) for x in locals_]).view(dtype) if p > 1 else as_bits(locals_[0]).clone().view(dtype)
    if p > 1 and counters is not None:
        _charge_allgather(counters, [b.numel() for b in locals_], p)
    return out


# -- threads as ranks (the reference harness, comm.py:156-284) ---------------


class _Slot:
    __slots__ = ("kind", "payloads", "results", "error", "done", "taken")

    def __init__(self, kind: str):
        self.kind = kind
        self.payloads: dict[int, object] = {}
        self.results: list | None = None
        self.error: BaseException | None = None
        self.done = False
        self.taken = 0


class WorkerGroup:
    """p ranks inside one process; the n-th collective call of every rank meets
    in slot n, the last arriver runs the device collective once (comm.py:168-258)."""

    def __init__(self, size: int, *, timeout: float = 30.0):
        if size < 1:
            raise ValueError("group size must be >= 1")
        self.size = size
        self.timeout = timeout
        self.counters = [CommCounters() for _ in range(size)]
        self._cond = threading.Condition()
        self._slots: dict[int, _Slot] = {}
        self._call_index = [0] * size

    def all_reduce_sum(self, rank: int, buf) -> None:
        self._collective(rank, "all_reduce_sum", buf)

    def all_reduce_sum_mixed(self, rank: int, buf, mode: PrecisionMode) -> None:
        self._collective(rank, f"all_reduce_sum_mixed:{mode.name}", (buf, mode))

    def all_gather(self, rank: int, local):
        return self._collective(rank, "all_gather", local)

    def barrier(self, rank: int) -> None:
        self._collective(rank, "barrier", None)

    def _collective(self, rank: int, kind: str, payload):
        if not 0 <= rank < self.size:
            raise CollectiveError(f"rank {rank} outside group of {self.size}")
        with self._cond:
            idx = self._call_index[rank]
            self._call_index[rank] += 1
            slot = self._slots.get(idx)
            if slot is None:
                slot = self._slots[idx] = _Slot(kind)
            elif slot.kind != kind and slot.error is None:
                slot.error = CollectiveError(
                    f"rank {rank} entered {kind!r} while others run {slot.kind!r}"
                )
                slot.done = True
                self._cond.notify_all()
            slot.payloads[rank] = payload
            if len(slot.payloads) == self.size and not slot.done:
                try:
                    slot.results = self._execute(kind, [slot.payloads[r] for r in range(self.size)])
                except BaseException as exc:  # noqa: BLE001 - forwarded to every rank
                    slot.error = exc
                slot.done = True
                self._cond.notify_all()
            else:
                deadline = time.monotonic() + self.timeout
                while not slot.done:
                    remaining = deadline - time.monotonic()
                    if remaining <= 0:
                        absent = sorted(set(range(self.size)) - set(slot.payloads))
                        slot.error = CollectiveTimeout(kind, absent)
                        slot.done = True
                        self._cond.notify_all()
                        break
                    self._cond.wait(remaining)
            error = slot.error
            results = slot.results
            slot.taken += 1
            if slot.taken == self.size:
                self._slots.pop(idx, None)
        if error is not None:
            raise error
        return results[rank] if results is not None else None

    def _execute(self, kind: str, payloads: list):
        if kind == "barrier":
            return None
        if kind == "all_reduce_sum":
            ring_all_reduce(payloads, self.counters)
            return None
        if kind.startswith("all_reduce_sum_mixed"):
            ring_all_reduce_mixed([p[0] for p in payloads], payloads[0][1], self.counters)
            return None
        if kind == "all_gather":
            out = ring_all_gather(payloads, self.counters)
            return [as_bits(out).clone().view(out.dtype) for _ in range(self.size)]
        raise CollectiveError(f"unknown collective {kind!r}")

    def run(self, fn, *args) -> list:
        """Drive fn(rank, *args) on every rank concurrently; re-raise the first
        real failure ahead of the timeouts it caused (comm.py:262-284)."""
        if self.size == 1:
            return [fn(0, *args)]
        results = [None] * self.size
        errors: list[BaseException | None] = [None] * self.size

        def body(r: int) -> None:
            try:
                results[r] = fn(r, *args)
            except BaseException as exc:  # noqa: BLE001
                errors[r] = exc

        threads = [threading.Thread(target=body, args=(r,), name=f"rank{r}") for r in range(self.size)]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        first = next((e for e in errors if e is not None and not isinstance(e, CollectiveTimeout)), None)
        first = first or next((e for e in errors if e is not None), None)
        if first is not None:
            raise first
        return results


# -- one process per GPU (torch.distributed over NCCL / NVLink) --------------


FoldFn = Callable[..., None]
ALGOS = ("exact", "nccl", "p2p", "fused")


def _wire(t: torch.Tensor) -> torch.Tensor:
    # collectives only move bytes; NCCL has no uint16, so brain travels as bf16
    return t.view(torch.bfloat16) if t.dtype == torch.uint16 else t


def _env_int(name: str, default: int, lo: int) -> int:
    raw = os.environ.get(name, "").strip()
    if not raw:
        return default
    try:
        val = int(raw)
    except ValueError:
        raise CollectiveError(f"{name}={raw!r} is not an integer") from None
    if val < lo:
        raise CollectiveError(f"{name}={val} must be >= {lo}")
    return val


# interleave assembly through the NVSwitch multicast mapping when the peer
# buffer has one and the group has at least this many ranks
# (TENVEC_B200_MULTICAST=0: always push to each peer)
_MULTICAST_MIN = _env_int("TENVEC_B200_MULTICAST", 3, 0)
# the per-peer push as one launch storing into every joint copy (A/B knob:
# TENVEC_B200_PUSH_ONE_LAUNCH=0 launches one repack per destination)
_PUSH_ONE_LAUNCH = os.environ.get("TENVEC_B200_PUSH_ONE_LAUNCH", "1") != "0"


@dataclass(frozen=True)
class FusedPlan:
    """Index math of the split-mode contraction fused with its reduction
    (RankGroup.tvc_reduce_fused) for a rank-local (u, n_k, v) view over p
    ranks.  The (u, v) output is cut into p owner ranges along u (whole slabs,
    u >= p) or along v (columns, u == 1); owner c receives every rank's
    partial sums of its range in p slots of ``slot_elems`` and keeps the
    folded range in slot p."""

    along_u: bool
    outer: int            # extent that is partitioned (u or v)
    q: int                # outer indices per owner (the last owner may hold fewer)
    unit: int             # output elements per outer index
    bounds: tuple         # per owner: [lo, hi) outer indices
    sizes: tuple          # per owner: output elements
    chunk: int            # output elements of a full owner range
    ring_chunk: int       # ring_chunks' chunk of the whole output (mixed fold order)
    slot_elems: int
    slot_bytes: int

    @property
    def n(self) -> int:
        return sum(self.sizes)


def fused_plan(u: int, v: int, p: int, storage_bytes: int) -> FusedPlan | None:
    """None when the view has no owner partition (p == 1, or 1 < u < p)."""
    if p == 1 or not (u >= p or u == 1):
        return None
    along_u = u >= p
    outer = u if along_u else v
    q = -(-outer // p)
    unit = v if along_u else 1
    bounds = tuple((min(c * q, outer), min((c + 1) * q, outer)) for c in range(p))
    sizes = tuple((b - a) * unit for a, b in bounds)
    chunk = q * unit
    ring = ring_chunks(u * v, p)
    slot_bytes = -(-chunk * storage_bytes // 16) * 16
    return FusedPlan(along_u, outer, q, unit, bounds, sizes, chunk, ring[0][1] - ring[0][0],
                     slot_bytes // storage_bytes, slot_bytes)


class RankGroup:
    """This process is rank ``rank`` of ``size``.  Same method names as
    ``WorkerGroup`` so the dtvc / dhopm3 rank bodies run unchanged; the rank
    argument must be this process's rank.

    ``transport`` moves the bytes (default ``TorchTransport``: torch.distributed
    over NCCL/NVLink plus symmetric memory; ``loopback.LoopbackTransport`` runs
    the same code as thread-ranks on one GPU).  ``fold`` is the local reduction
    (default: the tv_rank_fold kernel); CPU multi-process tests inject a host
    fold to exercise the chunk logic over gloo without a GPU.

    ``algo`` (default from TENVEC_B200_ALLREDUCE, else "fused"):
      exact  all-to-all of ring chunks + fold kernel + all-gather (NCCL moves
             the bytes), reference-exact;
      p2p    the same fold over PEER memory: every rank's buffer is mapped
             into its peers (NVLink), rank c folds ring chunk c straight from
             its peers' buffers with the fold kernel, a select kernel gathers
             the reduced chunks; three device barriers, no NCCL, reference-exact;
      nccl   ncclAllReduce (rank-consistent, not reference-ordered);
      fused  for dtvc's split-mode contraction (k == s): the TVC itself writes
             each owner's output range straight into that owner's receive slot
             in peer memory, the owner folds its p slots in the reference
             order, and every rank gathers the reduced ranges from its peers
             (``tvc_reduce_fused``); no NCCL, no partial written to local HBM
             first.  Other reductions run as "exact"; when any rank cannot map
             peer memory, every rank falls back to "exact" together.

    Failure semantics (comm.py:206-235, 279-284): collectives are numbered in
    issue order; ``timeout`` (default TENVEC_B200_TIMEOUT, else 300 s) bounds
    every device barrier (tv_peer_barrier records the missing ranks instead of
    hanging), every host collective and ``wait()``.  A timeout raises
    ``CollectiveTimeout(kind, absent)``, the absent ranks read from the device
    barrier's status or from a ledger of issued collectives in the store, and
    leaves the group failed.  ``check=True`` (or
    TENVEC_B200_CHECK_COLLECTIVES=1) also meets every rank in the store before
    each collective, raising CollectiveError on a kind mismatch the way the
    reference's rendezvous slot does (one store round trip per collective).
    """

    def __init__(self, group=None, *, algo: str | None = None, fold: FoldFn | None = None,
                 timeout: float | None = None, transport=None, check: bool | None = None):
        algo = algo or os.environ.get("TENVEC_B200_ALLREDUCE", "fused")
        if algo not in ALGOS:
            raise CollectiveError(f"unknown allreduce algorithm {algo!r}")
        self.t = transport if transport is not None else TorchTransport(group)
        self.group = group
        self.size = self.t.size
        self.rank = self.t.rank
        self.algo = algo
        self.fold = fold or device_fold_strided
        self.counters = [CommCounters() for _ in range(self.size)]
        if timeout is None:
            try:
                timeout = float(os.environ.get("TENVEC_B200_TIMEOUT", "300"))
            except ValueError:
                raise CollectiveError("TENVEC_B200_TIMEOUT must be a number of seconds") from None
        if timeout <= 0:
            raise CollectiveError("the collective timeout must be positive")
        self.timeout = float(timeout)
        self.check = (os.environ.get("TENVEC_B200_CHECK_COLLECTIVES", "0") == "1") if check is None else check
        self.assembly_path = None  # how the last interleave assembly moved its parts
        # streams of the fused reduction's owner launches (validated up front:
        # a bad value must not surface after a barrier has been enqueued)
        self.lanes = _env_int("TENVEC_B200_OWNER_LANES", 2, 1)
        self._lane_streams: tuple | None = None
        self._peer: PeerBuffer | None = None
        self._status: torch.Tensor | None = None  # tv_peer_barrier status block
        self._epoch_kind: dict[int, str] = {}
        self._issued = 0
        self._inflight: collections.deque = collections.deque()
        self._failed: CollectiveError | None = None

    # -- bookkeeping of issued collectives ------------------------------------
    def _begin(self, kind: str) -> int:
        if self._failed is not None:
            raise self._failed
        self._issued += 1
        seq = self._issued
        if self.check:
            absent, kinds = self.t.check_kind(self.rank, seq, kind, self.timeout)
            if absent:
                raise self._fail(CollectiveTimeout(kind, absent))
            other = sorted({k for k in kinds.values() if k != kind})
            if other:
                raise CollectiveError(f"rank {self.rank} entered {kind!r} while others run {other[0]!r}")
        return seq

    def _end(self, seq: int, kind: str, on_device: bool) -> None:
        if not on_device:
            return
        ev = torch.cuda.Event()
        ev.record()
        self._inflight.append((seq, kind, ev))
        while len(self._inflight) > 1 and self._inflight[0][2].query():
            self._inflight.popleft()
        if len(self._inflight) > 4096:
            self._inflight.popleft()

    def _fail(self, err: CollectiveError) -> CollectiveError:
        self._failed = err
        return err

    def _timed_out(self, seq: int, kind: str) -> CollectiveTimeout:
        absent = self.t.absent_ranks(self.rank, seq, self._issued, min(self.timeout, 5.0))
        self.t.abort()
        return self._fail(CollectiveTimeout(kind, absent if absent is not None else []))

    def _host(self, seq: int, kind: str, fn, *args) -> None:
        """Run one transport collective, mapping its failures."""
        try:
            fn(*args)
        except CollectiveTimeout as exc:
            raise self._fail(exc)
        except CollectiveError:
            raise
        except RuntimeError as exc:
            if self.t.is_timeout(exc):
                raise self._timed_out(seq, kind) from exc
            raise CollectiveError(f"{kind}: {exc}") from exc

    def wait(self, timeout: float | None = None) -> None:
        """Block until every collective this rank issued has completed on the
        device, giving up when none completes for ``timeout`` seconds
        (default: the group's).  Raises
        CollectiveTimeout naming the absent ranks when a device barrier gave
        up or a collective is still stuck at the deadline."""
        if self._failed is not None:
            raise self._failed
        limit = self.timeout if timeout is None else timeout
        deadline = time.monotonic() + limit
        while self._inflight:
            seq, kind, ev = self._inflight[0]
            if ev.query():
                self._inflight.popleft()
                deadline = time.monotonic() + limit  # progress: the clock restarts
                continue
            if time.monotonic() > deadline:
                raise self._timed_out(seq, kind)
            time.sleep(0.0005)
        self._check_status()

    def _check_status(self) -> None:
        if self._status is None:
            return
        st = self._status.cpu().tolist()
        if st[0] != 0:
            mask = (st[2] & 0xFFFFFFFF) | ((st[3] & 0xFFFFFFFF) << 32)
            absent = [r for r in range(self.size) if mask >> r & 1]
            raise self._fail(CollectiveTimeout(self._epoch_kind.get(st[1], "peer barrier"), absent))

    @contextlib.contextmanager
    def timeout_scope(self, timeout: float | None):
        """Temporarily use another timeout (dhopm3(timeout=...))."""
        if timeout is None:
            yield self
            return
        old = self.timeout
        self.timeout = float(timeout)
        try:
            yield self
        finally:
            self.timeout = old

    # -- peer memory -----------------------------------------------------------
    def _peer_buffer(self, nbytes: int, device) -> PeerBuffer:
        """This group's peer buffer with at least nbytes of data (collective
        when it has to grow; raises PeerMemoryUnavailable on every rank)."""
        if self._peer is not None and self._peer.capacity >= nbytes:
            return self._peer
        # the allocation synchronises every rank's device first, so nobody
        # still reads the buffer being replaced; every kernel is loaded before
        # the first barrier can spin
        with torch.cuda.device(device):
            _lib.preload()
        pb = self.t.peer_buffer(max(nbytes, 1 << 20), device)
        self._peer = pb
        self._epoch_kind.clear()
        if self._status is None:
            self._status = torch.zeros(4, dtype=torch.int32, device=device)
        return pb

    def _dev_barrier(self, pb: PeerBuffer, kind: str) -> None:
        pb.epoch += 1
        self._epoch_kind[pb.epoch] = kind
        if len(self._epoch_kind) > 4096:
            self._epoch_kind.pop(next(iter(self._epoch_kind)))
        lib = _lib.load()
        _lib.check(lib.tv_peer_barrier(pb.bases_arr, self.size, self.rank, pb.epoch,
                                       int(self.timeout * 1e9), self._status.data_ptr(),
                                       _lib.stream_ptr()), f"{kind}: barrier")

    def _reduce_p2p(self, buf: torch.Tensor, mixed: bool, mode: PrecisionMode | None,
                    sizes: list[int], seq: int) -> None:
        p, rank = self.size, self.rank
        n, sb = buf.numel(), buf.element_size()
        pb = self._peer_buffer(n * sb, buf.device)
        mine = as_bits(pb.local_data[: n * sb].view(as_bits(buf).dtype))
        mine.copy_(as_bits(buf))
        q = sizes[0]
        lib = _lib.load()
        st, ct = _pair_for(buf, mode)
        stream = _lib.stream_ptr()
        self._dev_barrier(pb, "allreduce")           # every partial is in place
        if sizes[rank]:
            off = rank * q * sb
            srcs = (ctypes.c_void_p * p)(*[pb.data(c) + off for c in range(p)])
            _lib.check(lib.tv_rank_fold(srcs, p, sizes[rank], 0, rank, st, ct, int(mixed),
                                        pb.data(rank) + off, stream), "p2p fold")
        self._dev_barrier(pb, "allreduce")           # every chunk is reduced
        srcs = (ctypes.c_void_p * p)(*[pb.data(c) for c in range(p)])
        _lib.check(lib.tv_rank_select(srcs, p, n, q, st, buf.data_ptr(), stream), "p2p gather")
        self._dev_barrier(pb, "allreduce")           # peers done reading this buffer
        self._end(seq, "allreduce", True)

    def _owner_streams(self, device) -> tuple:
        if self._lane_streams is None:
            self._lane_streams = tuple(torch.cuda.Stream(device=device) for _ in range(self.lanes))
        return self._lane_streams

    def tvc_reduce_fused(self, part, xv: torch.Tensor, k: int, mode: PrecisionMode,
                         counters: list[CommCounters] | None = None,
                         finish_stream: torch.cuda.Stream | None = None) -> torch.Tensor | None:
        """dtvc's split-mode contraction fused with its reduction over peer
        memory (algo="fused", geometry in ``fused_plan``): this rank's TVC
        launches write owner range c straight into rank c's receive slot for
        this rank (a peer pointer: the stores cross NVLink); after a device
        barrier each owner folds its p slots in the reference's per-element
        order (ascending rank, or the mixed ring's, comm.py:84-134), and after
        a second barrier every rank gathers the p reduced ranges from the
        owners.  The fold is the other transports' fold; the partial sums are
        those of a TVC over the owner's sub-range, which on integer data (the
        parity fills) are exact and on float data may round differently from
        a full-slab launch, within the TVC tolerance.  Returns the replicated
        output, or None when the view has no owner partition (1 < u < p) or
        peer memory is unavailable and the caller falls back.  With
        ``finish_stream`` the fold and gather run there (the caller waits on
        it before reading the output), overlapping later work."""
        from .kernels import launch_getvc, launch_tvc
        from .tensor import matricize_dims

        p, rank = self.size, self.rank
        md = matricize_dims(part.shape, k)
        nk, v = md.nk, md.v
        plan = fused_plan(md.u, v, p, mode.storage_bytes)
        if plan is None:
            return None
        seq = self._begin("dtvc_reduce")
        try:
            pb = self._peer_buffer((p + 1) * plan.slot_bytes, part.buf.device)
        except PeerMemoryUnavailable as exc:
            warnings.warn(f"RankGroup: {exc}; using algo='exact'")
            self.algo = "exact"
            self._issued -= 1  # the fallback issues its own collective
            return None
        sb = mode.storage_bytes
        counters = self.counters if counters is None else counters
        for cc in counters:
            cc.collective_calls += 1
        _charge_allreduce_movement(counters, list(ring_sizes(plan.n, p)), p)
        lib = _lib.load()
        st_, ct_ = mode.tv_storage, mode.tv_compute
        a_ptr = part.buf.data_ptr()
        self._dev_barrier(pb, "dtvc_reduce")  # peers are done with the previous call's slots
        # the p owner launches alternate over the lanes so one launch's tail
        # overlaps the next one's ramp (each is a full-GPU grid)
        main = torch.cuda.current_stream()
        lanes = self._owner_streams(part.buf.device)
        for ls in lanes:
            ls.wait_stream(main)
            xv.record_stream(ls)
        for j in range(p):  # own range first, then the peers in ring order
            c = (rank + j) % p
            lo, hi = plan.bounds[c]
            if hi <= lo:
                continue
            dst = pb.data(c) + rank * plan.slot_bytes
            lane = lanes[j % len(lanes)]
            if plan.along_u:
                launch_tvc(a_ptr + lo * nk * v * sb, mode, hi - lo, nk, v, xv.data_ptr(), 1.0, 0.0, dst,
                           part.buf.device, lane, "fused dtvc: contraction into peer memory")
            else:  # u == 1: columns [lo, hi) of the nk x v slab, a strided vecmat
                launch_getvc(1, a_ptr + lo * sb, mode, nk, hi - lo, v, xv.data_ptr(), 1.0, 0.0, dst,
                             part.buf.device, lane, "fused dtvc: contraction into peer memory")
        for ls in lanes:
            main.wait_stream(ls)
        out = torch.empty(plan.n, dtype=mode.torch_storage, device=part.buf.device)
        if finish_stream is not None:
            finish_stream.wait_stream(main)
            out.record_stream(finish_stream)
        with torch.cuda.stream(finish_stream or main):
            stream = _lib.stream_ptr()
            self._dev_barrier(pb, "dtvc_reduce")  # every slot holds its writer's partial range
            if plan.sizes[rank]:
                _lib.check(lib.tv_rank_fold_range(pb.data(rank), plan.slot_elems, p, plan.sizes[rank],
                                                  plan.ring_chunk, rank * plan.chunk, st_, ct_,
                                                  int(mode.mixed), pb.data(rank) + p * plan.slot_bytes,
                                                  stream), "fused dtvc: owner fold")
            self._dev_barrier(pb, "dtvc_reduce")  # every owner's reduced range is ready
            srcs = (ctypes.c_void_p * p)(*[pb.data(c) + p * plan.slot_bytes - c * plan.chunk * sb
                                           for c in range(p)])
            _lib.check(lib.tv_rank_select(srcs, p, plan.n, plan.chunk, st_, out.data_ptr(), stream),
                       "fused dtvc: gather")
            self._end(seq, "dtvc_reduce", True)
        return out

    def native_comm(self) -> int:
        """This rank's NCCL communicator for the C-ABI's distributed entry
        points (tv_comm_init_rank), created on first use: rank 0's unique id
        travels through the group's store.  One process per GPU only."""
        if getattr(self, "_native_comm", None):
            return self._native_comm
        store = getattr(self.t, "store", None)
        if store is None or getattr(self.t, "backend", "") != "nccl":
            raise CollectiveError("native collectives need one process per GPU over NCCL (a c10d store)")
        lib = _lib.load()
        key = f"tenvec_b200/{self.t.gid}/nccl_unique_id"
        if self.rank == 0:
            uid = ctypes.create_string_buffer(128)
            _lib.check(lib.tv_comm_get_unique_id(uid), "native comm")
            store.set(key, bytes(uid.raw))
        raw = store.get(key)
        comm = ctypes.c_void_p()
        _lib.check(lib.tv_comm_init_rank(ctypes.create_string_buffer(bytes(raw), 128), self.size, self.rank,
                                         ctypes.byref(comm)), "native comm")
        self._native_comm = comm.value
        return self._native_comm

    # -- host-ordered collectives ----------------------------------------------
    def _check_rank(self, rank: int) -> None:
        if rank != self.rank:
            raise CollectiveError(f"rank {rank} called from process rank {self.rank}")

    def barrier(self, rank: int) -> None:
        self._check_rank(rank)
        seq = self._begin("barrier")
        self._host(seq, "barrier", self.t.barrier)

    def _reduce(self, buf: torch.Tensor, mixed: bool, mode: PrecisionMode | None,
                counters: list[CommCounters] | None) -> None:
        p, rank = self.size, self.rank
        n = buf.numel()
        sizes = list(ring_sizes(n, p))
        counters = self.counters if counters is None else counters
        seq = self._begin("allreduce")
        for c in counters:
            c.collective_calls += 1
        _charge_allreduce_movement(counters, sizes, p)
        if p == 1:
            return
        t = self.t
        if self.algo == "nccl" and not mixed:
            self._host(seq, "allreduce", t.all_reduce, buf, "sum")
            self._end(seq, "allreduce", buf.is_cuda)
            return
        if self.algo == "p2p" and n * buf.element_size() * p > SMALL_GATHER_BYTES:
            try:
                self._reduce_p2p(buf, mixed, mode, sizes, seq)
                return
            except PeerMemoryUnavailable as exc:
                warnings.warn(f"RankGroup: {exc}; using algo='exact'")
                self.algo = "exact"
        if n * buf.element_size() * p <= SMALL_GATHER_BYTES:
            # latency-bound sizes (dHOPM3 vectors): one all-gather of every
            # rank's buffer, then each rank folds all ring chunks itself --
            # the same values in the same order, one NCCL call instead of two
            everyone = torch.empty(p * n, dtype=buf.dtype, device=buf.device)
            self._host(seq, "allreduce", t.all_gather_into_tensor, _wire(everyone), _wire(buf.contiguous()))
            self.fold(everyone, n, p, n, buf, mixed=mixed, mode=mode, start=0, chunk=sizes[0])
            self._end(seq, "allreduce", buf.is_cuda)
            return
        mine = sizes[rank]
        recv = torch.empty(p * mine, dtype=buf.dtype, device=buf.device)
        self._host(seq, "allreduce", t.all_to_all_single, _wire(recv), _wire(buf.contiguous()),
                   [mine] * p, sizes)
        q = sizes[0]
        padded = torch.empty(q, dtype=buf.dtype, device=buf.device)
        if mine:
            self.fold(recv, mine, p, mine, padded[:mine], mixed=mixed, mode=mode, start=rank)
        gathered = torch.empty(p * q, dtype=buf.dtype, device=buf.device)
        self._host(seq, "allreduce", t.all_gather_into_tensor, _wire(gathered), _wire(padded))
        # chunk c sits at [c*q, c*q + sizes[c]); only the tail is short, so the
        # first n gathered elements are the reduced buffer in order
        as_bits(buf).copy_(as_bits(gathered[:n]))
        self._end(seq, "allreduce", buf.is_cuda)

    def all_reduce_sum(self, rank: int, buf: torch.Tensor,
                       counters: list[CommCounters] | None = None) -> None:
        self._check_rank(rank)
        self._reduce(buf, False, None, counters)

    def all_reduce_sum_mixed(self, rank: int, buf: torch.Tensor, mode: PrecisionMode,
                             counters: list[CommCounters] | None = None) -> None:
        self._check_rank(rank)
        self._reduce(buf, True, mode, counters)

    def all_reduce_normalize(self, rank: int, buf: torch.Tensor, mode: PrecisionMode, dst: torch.Tensor,
                             norm_slot: torch.Tensor, status_slot: torch.Tensor | None,
                             counter: torch.Tensor, counters: list[CommCounters] | None = None) -> bool:
        """dHOPM3's reduction of an iteration's vector with the normalisation
        folded into the fold kernel's epilogue (tv_rank_fold_normalize):
        dst <- normalize(allreduce(buf)) with the same bits as all_reduce_sum
        (exact or mixed ring order) followed by normalize (hopm.py:320-330);
        buf is left as it was.  Latency-sized vectors only (the all-gather
        path); returns False, doing nothing, when the caller must run the
        unfused sequence."""
        self._check_rank(rank)
        p = self.size
        n = buf.numel()
        if p == 1 or n == 0 or not buf.is_cuda or self.fold is not device_fold_strided or \
                (self.algo == "nccl" and not mode.mixed) or n * buf.element_size() * p > SMALL_GATHER_BYTES:
            return False
        sizes = list(ring_sizes(n, p))
        counters = self.counters if counters is None else counters
        seq = self._begin("allreduce")
        for c in counters:
            c.collective_calls += 1
        _charge_allreduce_movement(counters, sizes, p)
        everyone = torch.empty(p * n, dtype=buf.dtype, device=buf.device)
        self._host(seq, "allreduce", self.t.all_gather_into_tensor, _wire(everyone), _wire(buf.contiguous()))
        lib = _lib.load()
        sp = status_slot.data_ptr() if status_slot is not None else None
        _lib.check(lib.tv_rank_fold_normalize(everyone.data_ptr(), n, p, n, sizes[0], mode.tv_storage,
                                              mode.tv_compute, int(mode.mixed), dst.data_ptr(),
                                              norm_slot.data_ptr(), sp, counter.data_ptr(),
                                              _lib.stream_ptr()), "allreduce + normalize")
        self._end(seq, "allreduce", True)
        return True

    def raw_all_gather(self, t: torch.Tensor) -> torch.Tensor:
        """Uncounted byte all-gather of equal-length tensors (bookkeeping checks)."""
        seq = self._begin("all_gather")
        src = t.contiguous().view(torch.uint8)
        out = torch.empty(self.size * src.numel(), dtype=torch.uint8, device=t.device)
        self._host(seq, "all_gather", self.t.all_gather_into_tensor, out, src)
        self._end(seq, "all_gather", out.is_cuda)
        return out.view(t.dtype)

    def all_gather_padded(self, rank: int, local: torch.Tensor, counts: list[int]) -> tuple[torch.Tensor, int]:
        """all_gather without the final compaction: rank r's part sits at
        [r * q, r * q + counts[r]) of the result, q = max(counts) (what the
        repack kernel reads)."""
        self._check_rank(rank)
        p = self.size
        seq = self._begin("all_gather")
        for c in self.counters:
            c.collective_calls += 1
        _charge_allgather(self.counters, counts, p)
        q = max(counts)
        padded = torch.empty(q, dtype=local.dtype, device=local.device)
        as_bits(padded[: local.numel()]).copy_(as_bits(local))
        gathered = torch.empty(p * q, dtype=local.dtype, device=local.device)
        if p == 1:
            as_bits(gathered).copy_(as_bits(padded))
            return gathered, q
        self._host(seq, "all_gather", self.t.all_gather_into_tensor, _wire(gathered), _wire(padded))
        self._end(seq, "all_gather", gathered.is_cuda)
        return gathered, q

    def repack_from_peers(self, local: torch.Tensor, plan, u: int, v: int, out: torch.Tensor) -> bool:
        """The "interleave" assembly across processes: every rank PUSHES its
        part's runs straight into every rank's joint copy in peer memory
        (tv_repack_part; NVLink stores are posted, loads would pay a round
        trip each) -- from _MULTICAST_MIN ranks on, once, through the
        buffer's NVSwitch multicast address (tv_repack_part_multicast) -- then
        copies its own joint copy out; no NCCL.  Each rank picks its own way
        (alignment, an empty part); the parts land in the same places either
        way.  False (nothing done) when peer memory is not in use."""
        if self.size == 1 or self.algo not in ("fused", "p2p") or not local.is_cuda:
            return False
        p = self.size
        eb = local.element_size()
        nbytes = out.numel() * eb
        seq = self._begin("all_gather")
        try:
            pb = self._peer_buffer(nbytes, local.device)
        except PeerMemoryUnavailable as exc:
            warnings.warn(f"RankGroup: {exc}; using algo='exact'")
            self.algo = "exact"
            self._issued -= 1
            return False
        for c in self.counters:
            c.collective_calls += 1
        _charge_allgather(self.counters, [(b - a) * u * v for a, b in plan.ranges], p)
        self._dev_barrier(pb, "all_gather")  # every rank is done with its joint copy's previous contents
        lib = _lib.load()
        stream = _lib.stream_ptr()
        # two ranks: the push writes its own copy locally and sends one over
        # NVLink, the multicast would send both; from three on it saves p - 2
        # copies of this GPU's egress (C3 at N = 4: 11.8 -> 9.6 ms per step)
        mc = pb.mc + TV_PEER_HEADER if pb.mc and _MULTICAST_MIN and p >= _MULTICAST_MIN else 0
        ext = min(plan.chunk, plan.extent - self.rank * plan.chunk)
        if mc and ext > 0 and (local.data_ptr() | mc | plan.chunk * v * eb | ext * v * eb
                               | plan.extent * v * eb) % 16 == 0:
            # one store per unit through the NVSwitch multicast mapping
            _lib.check(lib.tv_repack_part_multicast(local.data_ptr(), self.rank, p, u, plan.extent, v,
                                                    plan.chunk, eb, mc, stream), "interleave assembly")
            self.assembly_path = "multicast"
        elif ext > 0 and _PUSH_ONE_LAUNCH and (local.data_ptr() | plan.chunk * v * eb | ext * v * eb
                                               | plan.extent * v * eb) % 16 == 0 \
                and all(pb.data(c) % 16 == 0 for c in range(p)):
            # one launch stores every unit into all p joint copies
            dsts = (ctypes.c_void_p * p)(*[pb.data((self.rank + j) % p) for j in range(p)])
            _lib.check(lib.tv_repack_part_peers(local.data_ptr(), self.rank, p, u, plan.extent, v, plan.chunk, eb,
                                                dsts, p, stream), "interleave assembly")
            self.assembly_path = "push"
        else:
            self.assembly_path = "push"
            for j in range(p):  # own copy first, then the peers in ring order
                c = (self.rank + j) % p
                _lib.check(lib.tv_repack_part(local.data_ptr(), self.rank, p, u, plan.extent, v, plan.chunk, eb,
                                              pb.data(c), stream), "interleave assembly")
        self._dev_barrier(pb, "all_gather")  # every part has landed in every joint copy
        out.view(torch.uint8).copy_(pb.local_data[:nbytes]) if out.dtype != torch.uint16 else \
            out.view(torch.int16).view(torch.uint8).copy_(pb.local_data[:nbytes])
        self._end(seq, "all_gather", True)
        return True

    def all_gather(self, rank: int, local: torch.Tensor, counts: list[int] | None = None
                   ) -> torch.Tensor:
        """Rank-order concatenation; ``counts`` gives every rank's length when
        they differ (the last rank of a split is usually short)."""
        self._check_rank(rank)
        p = self.size
        seq = self._begin("all_gather")
        for c in self.counters:
            c.collective_calls += 1
        if counts is None:
            counts = [local.numel()] * p
        _charge_allgather(self.counters, counts, p)
        if p == 1:
            return as_bits(local).clone().view(local.dtype)
        q = max(counts)
        padded = torch.empty(q, dtype=local.dtype, device=local.device)
        as_bits(padded[: local.numel()]).copy_(as_bits(local))
        gathered = torch.empty(p * q, dtype=local.dtype, device=local.device)
        self._host(seq, "all_gather", self.t.all_gather_into_tensor, _wire(gathered), _wire(padded))
        self._end(seq, "all_gather", gathered.is_cuda)
        if all(c == q for c in counts):
            return gathered
        parts = [gathered[r * q: r * q + counts[r]] for r in range(p)]
        return torch.cat([as_bits(x) for x in parts]).view(local.dtype)
