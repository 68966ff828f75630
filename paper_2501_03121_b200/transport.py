"""What RankGroup needs from the machinery that connects its ranks.

``RankGroup`` (comm.py) holds the reference's collective semantics
(pkg/src/tenvec/comm.py:58-284): which values are folded in which order, the
counters, the timeout and error rules.  The transport only moves bytes and
maps memory:

* host-ordered collectives on device tensors (all-gather, all-to-all,
  all-reduce, barrier), enqueued on the caller's current stream;
* a peer buffer per rank -- every rank's buffer mapped into this process
  (NVLink peer memory across GPUs), whose first ``TV_PEER_HEADER`` bytes hold
  the arrival words of ``tv_peer_barrier``;
* a ledger to name the ranks that never arrived when a collective times out
  (the reference's ``CollectiveTimeout(kind, absent)``, comm.py:226-235).

``TorchTransport`` is the production one: torch.distributed (NCCL over
NVLink / NVSwitch between the GPUs of a box, gloo on CPU) plus torch
symmetric memory for the peer buffers and the c10d store for the ledger.
``loopback.LoopbackTransport`` runs p ranks as threads on ONE GPU with the
same interface, so the multi-GPU code paths are exercised bit for bit on a
single device.
"""

from __future__ import annotations

import ctypes
import datetime
import itertools
import warnings

import torch

from ._lib import TV_PEER_HEADER
from .errors import CollectiveError

__all__ = ["PeerBuffer", "PeerMemoryUnavailable", "TorchTransport", "TV_PEER_HEADER"]


class PeerMemoryUnavailable(CollectiveError):
    """Some rank of the group could not map peer memory; every rank falls back
    together (the decision is collective)."""


class PeerBuffer:
    """One rank's share of a peer-mapped allocation plus every rank's base
    address as mapped in this process.  Data starts TV_PEER_HEADER bytes in;
    the header holds the barrier words (zero on creation)."""

    __slots__ = ("local", "bases", "capacity", "epoch", "bases_arr", "keep", "mc")

    def __init__(self, local: torch.Tensor, bases: list[int], keep=None, mc: int = 0):
        self.local = local
        self.bases = [int(b) for b in bases]
        # NVSwitch multicast address of the same bytes in every rank's buffer
        # (a store there lands in all of them), 0 when the fabric has none
        self.mc = int(mc)
        self.capacity = local.numel() - TV_PEER_HEADER
        self.epoch = 0
        self.bases_arr = (ctypes.c_void_p * len(self.bases))(*self.bases)
        self.keep = keep  # whatever keeps the mapping alive (handles, peer tensors)

    def data(self, rank: int) -> int:
        """Device address of rank's data region, as mapped here."""
        return self.bases[rank] + TV_PEER_HEADER

    @property
    def local_data(self) -> torch.Tensor:
        return self.local[TV_PEER_HEADER:]


_OPS = {"sum": "SUM", "max": "MAX", "min": "MIN"}
_GROUP_IDS = itertools.count()


class TorchTransport:
    """torch.distributed + symmetric memory (one process per GPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise CollectiveError("torch.distributed is not initialised")
        self._dist = dist
        self.group = group
        self.size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = str(dist.get_backend(group))
        # every process builds its RankGroups in the same order: a shared id
        self.gid = next(_GROUP_IDS)
        try:
            from torch.distributed.distributed_c10d import _get_default_store

            self.store = _get_default_store()
        except Exception:  # noqa: BLE001 - no ledger: absent ranks reported as unknown
            self.store = None

    # -- host-ordered collectives ---------------------------------------------
    def all_gather_into_tensor(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        self._dist.all_gather_into_tensor(out, inp, group=self.group)

    def all_to_all_single(self, out: torch.Tensor, inp: torch.Tensor, out_splits: list[int],
                          in_splits: list[int]) -> None:
        self._dist.all_to_all_single(out, inp, output_split_sizes=out_splits,
                                     input_split_sizes=in_splits, group=self.group)

    def all_reduce(self, t: torch.Tensor, op: str = "sum") -> None:
        self._dist.all_reduce(t, op=getattr(self._dist.ReduceOp, _OPS[op]), group=self.group)

    def barrier(self) -> None:
        self._dist.barrier(group=self.group)

    # -- peer memory ---------------------------------------------------------
    def peer_buffer(self, nbytes: int, device) -> PeerBuffer:
        """A new symmetric allocation of TV_PEER_HEADER + nbytes per rank.
        Collective, and so is the verdict: if any rank fails to allocate or
        map it, every rank raises PeerMemoryUnavailable."""
        import torch.distributed._symmetric_memory as symm_mem

        name = (self.group or self._dist.group.WORLD).group_name
        t, err = None, None
        try:
            with warnings.catch_warnings():  # deprecated (and unnecessary) from torch 2.11 on
                warnings.simplefilter("ignore", FutureWarning)
                symm_mem.enable_symm_mem_for_group(name)
            t = symm_mem.empty(TV_PEER_HEADER + nbytes, dtype=torch.uint8, device=device)
            t[:TV_PEER_HEADER].zero_()
        except Exception as exc:  # noqa: BLE001
            err = exc
        self._agree(err is None, device, "allocate", err)
        hdl, err = None, None
        try:
            hdl = symm_mem.rendezvous(t, name)
        except Exception as exc:  # noqa: BLE001
            err = exc
        self._agree(err is None, device, "map", err)
        torch.cuda.synchronize(device)  # headers are zero before any peer posts
        self.barrier()
        bases = [int(p) for p in hdl.buffer_ptrs]
        mc = 0
        try:  # only when the multicast mapping provably starts where our tensor does
            if int(getattr(hdl, "offset", 0)) == 0 and bases[self.rank] == t.data_ptr():
                mc = int(hdl.multicast_ptr or 0)
        except Exception:  # noqa: BLE001 - no multicast object: unicast pushes
            mc = 0
        return PeerBuffer(t, bases, keep=hdl, mc=mc)

    def _agree(self, ok: bool, device, what: str, err) -> None:
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                            device=device if self.backend == "nccl" else "cpu")
        self.all_reduce(flag, "min")
        if int(flag.item()) == 0:
            why = f"{err!r:.200}" if err is not None else "failed on another rank"
            raise PeerMemoryUnavailable(f"peer memory: {what} {why}")

    # -- ledger / failure handling -------------------------------------------
    def absent_ranks(self, rank: int, seq: int, issued: int, grace: float) -> list[int] | None:
        """Publish how many collectives this rank has issued and read everyone
        else's: the ranks that never issued collective ``seq`` are absent.
        None when there is no store to ask."""
        if self.store is None:
            return None
        prefix = f"tenvec_b200/{self.gid}/issued/"
        try:
            self.store.set(prefix + str(rank), str(issued))
        except Exception:  # noqa: BLE001
            return None
        absent = []
        for r in range(self.size):
            if r == rank:
                continue
            try:
                self.store.wait([prefix + str(r)], datetime.timedelta(seconds=max(grace, 0.01)))
                got = int(self.store.get(prefix + str(r)))
            except Exception:  # noqa: BLE001 - never published: gone or stuck elsewhere
                got = -1
            if got < seq:
                absent.append(r)
        return absent

    def check_kind(self, rank: int, seq: int, kind: str, timeout: float) -> tuple[list[int], dict]:
        """Strict mode: meet every rank at collective ``seq`` through the store
        before touching the device (the reference's rendezvous slot,
        comm.py:206-216).  Returns (absent ranks, {rank: kind})."""
        if self.store is None:
            return [], {}
        prefix = f"tenvec_b200/{self.gid}/kind/{seq}/"
        self.store.set(prefix + str(rank), kind)
        kinds, absent = {rank: kind}, []
        for r in range(self.size):
            if r == rank:
                continue
            try:
                self.store.wait([prefix + str(r)], datetime.timedelta(seconds=max(timeout, 0.01)))
                kinds[r] = self.store.get(prefix + str(r)).decode()
            except Exception:  # noqa: BLE001
                absent.append(r)
        return absent, kinds

    def abort(self) -> None:
        """Best effort: tear the communicator down so kernels stuck on a dead
        peer return (the group is unusable afterwards)."""
        if self.backend != "nccl":  # gloo collectives already returned with the error
            return
        try:
            from torch.distributed.distributed_c10d import _abort_process_group

            _abort_process_group(self.group)
        except Exception:  # noqa: BLE001
            pass

    @staticmethod
    def is_timeout(exc: BaseException) -> bool:
        msg = str(exc).lower()
        return any(w in msg for w in ("timed out", "timeout", "connection closed", "connection reset",
                                      "broken pipe", "aborted"))
