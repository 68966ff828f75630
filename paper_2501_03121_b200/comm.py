"""Collectives: reference ring semantics on device buffers, in one process or
across processes.

Mirrors pkg/src/tenvec/comm.py:1-284 with two transports:

* In-process (every rank's buffer lives in this process, as in the
  reference): ``ring_all_reduce`` / ``ring_all_reduce_mixed`` run ONE fold
  kernel over the p device buffers (``tv_rank_fold``) that replays the
  reference's value order -- the ascending-rank sum (comm.py:95-97) or the
  mixed ring where chunk c starts at rank c and each hop computes
  demote(promote + promote) (comm.py:123-130) -- so results are bit-equal to
  the reference.  ``WorkerGroup`` keeps the threads-as-ranks rendezvous
  (comm.py:168-284) on top of them.

* One process per GPU (``RankGroup``, torch.distributed over NCCL/NVLink):
  the same values from an all-to-all of ring chunks (chunk c of every rank
  lands on rank c, in the storage format, i.e. reduced precision on the wire
  for the mixed modes), the same fold kernel on rank c, and an all-gather of
  the folded chunks.  Traffic equals a ring allreduce's reduce-scatter +
  all-gather; the result is bit-identical to the reference and to every other
  rank.  ``algo="nccl"`` uses ncclAllReduce instead (faster for huge
  buffers, rank-consistent but not reference-ordered).

Counters follow the reference's ring accounting (comm.py:64-81).
"""

from __future__ import annotations

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

__all__ = [
    "CollectiveError", "CollectiveTimeout", "CommCounters", "ring_chunks", "ring_all_reduce",
    "ring_all_reduce_mixed", "ring_all_gather", "WorkerGroup", "RankGroup", "device_fold",
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


def _wire(t: torch.Tensor) -> torch.Tensor:
    # collectives only move bytes; NCCL has no uint16, so brain travels as bf16
    return t.view(torch.bfloat16) if t.dtype == torch.uint16 else t


class RankGroup:
    """This process is rank ``rank`` of ``size`` (torch.distributed).  Same
    method names as ``WorkerGroup`` so the dtvc / dhopm3 rank bodies run
    unchanged; the rank argument must be this process's rank.

    ``fold`` is the local reduction (default: the tv_rank_fold kernel); CPU
    multi-process tests inject a host fold to exercise the chunk logic over
    gloo without a GPU.

    ``algo`` (default from TENVEC_B200_ALLREDUCE, else "fused"):
      exact  all-to-all of ring chunks + fold kernel + all-gather (NCCL moves
             the bytes), reference-exact;
      p2p    the same fold over PEER memory: every rank's buffer is a
             symmetric-memory allocation (torch symm_mem, NVLink mapped), rank c
             folds ring chunk c straight from its peers' buffers with the fold
             kernel, a select kernel gathers the reduced chunks; three device
             barriers, no NCCL, reference-exact;
      nccl   ncclAllReduce (rank-consistent, not reference-ordered);
      fused  for dtvc's split-mode contraction (k == s): the TVC itself writes
             each owner's output range straight into that owner's receive slot
             in peer (symmetric) memory over NVLink, the owner folds its p
             slots in the reference order, and every rank gathers the reduced
             ranges from its peers (``tvc_reduce_fused``); no NCCL, no partial
             written to local HBM first.  Other reductions run as "exact";
             without symmetric memory the group falls back to "exact".
    """

    def __init__(self, group=None, *, algo: str | None = None, fold: FoldFn | None = None):
        import os

        import torch.distributed as dist

        if not dist.is_initialized():
            raise CollectiveError("torch.distributed is not initialised")
        algo = algo or os.environ.get("TENVEC_B200_ALLREDUCE", "fused")
        if algo not in ("exact", "nccl", "p2p", "fused"):
            raise CollectiveError(f"unknown allreduce algorithm {algo!r}")
        self._dist = dist
        self.group = group
        self.size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.algo = algo
        self.fold = fold or device_fold_strided
        self.counters = [CommCounters() for _ in range(self.size)]
        self._sym = None  # (uint8 symmetric tensor, handle)

    # -- peer memory (algo="p2p") ---------------------------------------------
    def _symmetric(self, nbytes: int, device) -> tuple[torch.Tensor, object]:
        import torch.distributed._symmetric_memory as symm_mem

        if self._sym is None or self._sym[0].numel() < nbytes:
            name = (self.group or self._dist.group.WORLD).group_name
            try:
                symm_mem.enable_symm_mem_for_group(name)
            except Exception:  # noqa: BLE001 - newer torch enables groups lazily
                pass
            cap = max(nbytes, 1 << 20)
            t = symm_mem.empty(cap, dtype=torch.uint8, device=device)
            self._sym = (t, symm_mem.rendezvous(t, name))
        return self._sym

    def _reduce_p2p(self, buf: torch.Tensor, mixed: bool, mode: PrecisionMode | None,
                    sizes: list[int]) -> None:
        p, rank = self.size, self.rank
        n, sb = buf.numel(), buf.element_size()
        sym, hdl = self._symmetric(n * sb, buf.device)
        mine = as_bits(sym[: n * sb].view(as_bits(buf).dtype))
        mine.copy_(as_bits(buf))
        ptrs = [int(ptr) for ptr in hdl.buffer_ptrs]
        q = sizes[0]
        lib = _lib.load()
        st, ct = _pair_for(buf, mode)
        stream = _lib.stream_ptr()
        hdl.barrier(channel=0)                      # every partial is in place
        if sizes[rank]:
            off = rank * q * sb
            srcs = (ctypes.c_void_p * p)(*[ptr + off for ptr in ptrs])
            _lib.check(lib.tv_rank_fold(srcs, p, sizes[rank], 0, rank, st, ct, int(mixed),
                                        ptrs[rank] + off, stream), "p2p fold")
        hdl.barrier(channel=0)                      # every chunk is reduced
        srcs = (ctypes.c_void_p * p)(*ptrs)
        _lib.check(lib.tv_rank_select(srcs, p, n, q, st, buf.data_ptr(), stream), "p2p gather")
        hdl.barrier(channel=0)                      # peers done reading this buffer

    def _owner_streams(self, device) -> tuple:
        if getattr(self, "_lanes", None) is None:
            n = int(os.environ.get("TENVEC_B200_OWNER_LANES", "2"))
            self._lanes = tuple(torch.cuda.Stream(device=device) for _ in range(max(1, n)))
        return self._lanes

    def tvc_reduce_fused(self, part, xv: torch.Tensor, k: int, mode: PrecisionMode,
                         counters: list[CommCounters] | None = None,
                         finish_stream: torch.cuda.Stream | None = None) -> torch.Tensor | None:
        """dtvc's split-mode contraction fused with its reduction over peer
        memory (algo="fused").  The (u, n_k, v) output is cut into p owner
        ranges -- slab ranges when u >= p, column ranges when u == 1 -- and
        this rank's TVC launches write range c directly into rank c's receive
        slot for this rank (a peer pointer: the stores cross NVLink).  After a
        device barrier the owner folds its p slots (ascending rank / the mixed
        ring's per-element order, comm.py:84-134, the same bits as every other
        algorithm), and after a second barrier every rank gathers the p reduced
        ranges from the owners.  Returns the replicated output, or None when
        the view has no owner partition (1 < u < p) and the caller falls back.
        With ``finish_stream`` the fold and gather run there (the caller waits
        on it before reading the output), overlapping later work."""
        from .tensor import matricize_dims

        p, rank = self.size, self.rank
        md = matricize_dims(part.shape, k)
        u, nk, v = md.u, md.nk, md.v
        n = u * v
        if p == 1 or not (u >= p or u == 1):
            return None
        sb = mode.storage_bytes
        along_u = u >= p
        outer = u if along_u else v
        q = -(-outer // p)  # owner c holds outer indices [c q, (c+1) q)
        unit = v if along_u else 1  # output elements per outer index
        chunk = q * unit  # output elements per owner (the last one may be short)
        bounds = [(min(c * q, outer), min((c + 1) * q, outer)) for c in range(p)]
        sizes = [(b - a) * unit for a, b in bounds]
        ring = ring_chunks(n, p)
        slot_bytes = -(-chunk * sb // 16) * 16
        try:
            sym, hdl = self._symmetric((p + 1) * slot_bytes, part.buf.device)
        except Exception as exc:  # noqa: BLE001 - no symmetric memory here: NCCL transport
            warnings.warn(f"RankGroup: peer memory unavailable ({exc!r:.200}); using algo='exact'")
            self.algo = "exact"
            return None
        counters = self.counters if counters is None else counters
        for cc in counters:
            cc.collective_calls += 1
        _charge_allreduce_movement(counters, [b - a for a, b in ring], p)
        ptrs = [int(ptr) for ptr in hdl.buffer_ptrs]
        lib = _lib.load()
        st_, ct_ = mode.tv_storage, mode.tv_compute
        a_ptr = part.buf.data_ptr()
        hdl.barrier(channel=0)  # peers are done with the previous call's slots
        # the p owner launches alternate over two streams so one launch's tail
        # overlaps the next one's ramp (each is a full-GPU grid)
        main = torch.cuda.current_stream()
        lanes = self._owner_streams(part.buf.device)
        for ls in lanes:
            ls.wait_stream(main)
        for ls in lanes:
            xv.record_stream(ls)
        for j in range(p):  # own range first, then the peers in ring order
            c = (rank + j) % p
            lo, hi = bounds[c]
            if hi <= lo:
                continue
            dst = ptrs[c] + rank * slot_bytes
            ls = _lib.stream_ptr(lanes[j % len(lanes)])
            if along_u:
                rc = lib.tv_tvc(a_ptr + lo * nk * v * sb, st_, ct_, hi - lo, nk, v, xv.data_ptr(),
                                1.0, 0.0, dst, ls)
            else:  # u == 1: columns [lo, hi) of the nk x v slab, a strided vecmat
                rc = lib.tv_getvc(1, a_ptr + lo * sb, st_, ct_, nk, hi - lo, v, xv.data_ptr(),
                                  1.0, 0.0, dst, ls)
            _lib.check(rc, "fused dtvc: contraction into peer memory")
        for ls in lanes:
            main.wait_stream(ls)
        out = torch.empty(n, dtype=mode.torch_storage, device=part.buf.device)
        if finish_stream is not None:
            finish_stream.wait_stream(torch.cuda.current_stream())
            out.record_stream(finish_stream)
        with torch.cuda.stream(finish_stream or torch.cuda.current_stream()):
            stream = _lib.stream_ptr()
            hdl.barrier(channel=0)  # every slot holds its writer's partial range
            mine = sizes[rank]
            if mine:
                _lib.check(lib.tv_rank_fold_range(sym.data_ptr(), slot_bytes // sb, p, mine,
                                                  ring[0][1] - ring[0][0], rank * chunk, st_, ct_,
                                                  int(mode.mixed), sym.data_ptr() + p * slot_bytes,
                                                  stream), "fused dtvc: owner fold")
            hdl.barrier(channel=0)  # every owner's reduced range is ready
            srcs = (ctypes.c_void_p * p)(*[ptrs[c] + p * slot_bytes - c * chunk * sb for c in range(p)])
            _lib.check(lib.tv_rank_select(srcs, p, n, chunk, st_, out.data_ptr(), stream),
                       "fused dtvc: gather")
        return out

    def _check_rank(self, rank: int) -> None:
        if rank != self.rank:
            raise CollectiveError(f"rank {rank} called from process rank {self.rank}")

    def barrier(self, rank: int) -> None:
        self._check_rank(rank)
        self._dist.barrier(group=self.group)

    def _reduce(self, buf: torch.Tensor, mixed: bool, mode: PrecisionMode | None,
                counters: list[CommCounters] | None) -> None:
        p, rank, dist = self.size, self.rank, self._dist
        n = buf.numel()
        chunks = ring_chunks(n, p)
        sizes = [b - a for a, b in chunks]
        counters = self.counters if counters is None else counters
        for c in counters:
            c.collective_calls += 1
        _charge_allreduce_movement(counters, sizes, p)
        if p == 1:
            return
        if self.algo == "nccl" and not mixed:
            dist.all_reduce(buf, group=self.group)
            return
        if self.algo == "p2p" and n * buf.element_size() * p > SMALL_GATHER_BYTES:
            self._reduce_p2p(buf, mixed, mode, sizes)
            return
        if n * buf.element_size() * p <= SMALL_GATHER_BYTES:
            # latency-bound sizes (dHOPM3 vectors): one all-gather of every
            # rank's buffer, then each rank folds all ring chunks itself --
            # the same values in the same order, one NCCL call instead of two
            everyone = torch.empty(p * n, dtype=buf.dtype, device=buf.device)
            dist.all_gather_into_tensor(_wire(everyone), _wire(buf.contiguous()), group=self.group)
            self.fold(everyone, n, p, n, buf, mixed=mixed, mode=mode, start=0, chunk=sizes[0])
            return
        mine = sizes[rank]
        recv = torch.empty(p * mine, dtype=buf.dtype, device=buf.device)
        dist.all_to_all_single(_wire(recv), _wire(buf.contiguous()), output_split_sizes=[mine] * p,
                               input_split_sizes=sizes, group=self.group)
        q = sizes[0]
        padded = torch.empty(q, dtype=buf.dtype, device=buf.device)
        if mine:
            self.fold(recv, mine, p, mine, padded[:mine], mixed=mixed, mode=mode, start=rank)
        gathered = torch.empty(p * q, dtype=buf.dtype, device=buf.device)
        dist.all_gather_into_tensor(_wire(gathered), _wire(padded), group=self.group)
        # chunk c sits at [c*q, c*q + sizes[c]); only the tail is short, so the
        # first n gathered elements are the reduced buffer in order
        as_bits(buf).copy_(as_bits(gathered[:n]))

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
        sizes = [b - a for a, b in ring_chunks(n, p)]
        counters = self.counters if counters is None else counters
        for c in counters:
            c.collective_calls += 1
        _charge_allreduce_movement(counters, sizes, p)
        everyone = torch.empty(p * n, dtype=buf.dtype, device=buf.device)
        self._dist.all_gather_into_tensor(_wire(everyone), _wire(buf.contiguous()), group=self.group)
        lib = _lib.load()
        sp = status_slot.data_ptr() if status_slot is not None else None
        _lib.check(lib.tv_rank_fold_normalize(everyone.data_ptr(), n, p, n, sizes[0], mode.tv_storage,
                                              mode.tv_compute, int(mode.mixed), dst.data_ptr(),
                                              norm_slot.data_ptr(), sp, counter.data_ptr(),
                                              _lib.stream_ptr()), "allreduce + normalize")
        return True

    def raw_all_gather(self, t: torch.Tensor) -> torch.Tensor:
        """Uncounted byte all-gather of equal-length tensors (bookkeeping checks)."""
        src = t.contiguous().view(torch.uint8)
        out = torch.empty(self.size * src.numel(), dtype=torch.uint8, device=t.device)
        self._dist.all_gather_into_tensor(out, src, group=self.group)
        return out.view(t.dtype)

    def all_gather(self, rank: int, local: torch.Tensor, counts: list[int] | None = None
                   ) -> torch.Tensor:
        """Rank-order concatenation; ``counts`` gives every rank's length when
        they differ (the last rank of a split is usually short)."""
        self._check_rank(rank)
        p = self.size
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
        self._dist.all_gather_into_tensor(_wire(gathered), _wire(padded), group=self.group)
        if all(c == q for c in counts):
            return gathered
        parts = [gathered[r * q: r * q + counts[r]] for r in range(p)]
        return torch.cat([as_bits(x) for x in parts]).view(local.dtype)
