"""p ranks as threads on ONE GPU, driving the one-process-per-GPU code.

The reference runs its ranks as threads of one process
(pkg/src/tenvec/comm.py:168-284).  ``LoopbackWorld`` does the same for
``RankGroup``: each thread-rank gets its own CUDA stream and a
``LoopbackTransport`` with TorchTransport's interface, so the transports that
normally span GPUs -- "fused" (the split-mode TVC writing owner ranges into
peer slots), "p2p" and "exact" -- and dHOPM3's fold-and-normalise run
unchanged, with the same kernels, the same device barrier (tv_peer_barrier)
and the same index math, on a single device.  Peer buffers are ordinary
device allocations of the same GPU shared through the world.

Host-ordered collectives are emulated in stream order: every rank records an
event when its input is ready, the ranks meet on the host (a rendezvous slot
per call, with the reference's timeout and kind checks), each rank's stream
waits for its peers' events and copies, and a second meeting keeps inputs
alive until every peer has read them.

Two rules keep p ranks on one GPU from deadlocking on the spinning device
barrier: host waits poll an event (``_lib.host_wait``) instead of blocking in
the driver, and every stream gets its own hardware queue --
CUDA_DEVICE_MAX_CONNECTIONS (default 8) must cover the ranks' streams (about
5 per rank: its own, two owner lanes, two side streams), so set it to 32
before the CUDA context exists (tests/conftest.py does).

Used by the ``-m gpu`` tests to cover the multi-GPU transports on a one-GPU
box; also a debugging tool (a p-rank run needs one GPU).
"""

from __future__ import annotations

import os
import threading
import time
import warnings

import torch

from . import _lib
from .errors import CollectiveError, CollectiveTimeout
from .transport import TV_PEER_HEADER, PeerBuffer, PeerMemoryUnavailable

__all__ = ["LoopbackWorld", "LoopbackTransport"]


class _Meet:
    __slots__ = ("kind", "payloads", "error", "done", "taken")

    def __init__(self, kind: str):
        self.kind = kind
        self.payloads: dict[int, object] = {}
        self.error: BaseException | None = None
        self.done = False
        self.taken = 0


class LoopbackWorld:
    """Shared state of p thread-ranks on one device."""

    def __init__(self, size: int, device=None, *, timeout: float = 60.0, fail_peer_rank: int | None = None):
        if size < 1:
            raise ValueError("world size must be >= 1")
        self.size = size
        self.device = torch.device(device or "cuda", torch.cuda.current_device()) \
            if device is None or isinstance(device, str) else device
        self.timeout = timeout
        self.fail_peer_rank = fail_peer_rank  # test hook: this rank cannot map peer memory
        self._cond = threading.Condition()
        self._meets: dict[int, _Meet] = {}
        self._calls = [0] * size
        self.issued = [0] * size  # collectives issued per rank (the ledger)
        conns = int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8") or 8)
        if 5 * size > conns:
            warnings.warn(f"LoopbackWorld({size}): CUDA_DEVICE_MAX_CONNECTIONS={conns} < {5 * size}; "
                          "streams of different thread-ranks may share a hardware queue and a device "
                          "barrier can then wait for work queued behind it (set it to 32 before CUDA starts)")

    def transport(self, rank: int) -> "LoopbackTransport":
        return LoopbackTransport(self, rank)

    # -- host rendezvous -------------------------------------------------------
    def meet(self, rank: int, kind: str, payload, timeout: float | None = None) -> list:
        """The n-th meet of every rank shares slot n; returns every rank's
        payload.  Kind mismatch -> CollectiveError, a missing rank ->
        CollectiveTimeout(kind, absent) (comm.py:206-235)."""
        timeout = self.timeout if timeout is None else timeout
        with self._cond:
            idx = self._calls[rank]
            self._calls[rank] += 1
            m = self._meets.get(idx)
            if m is None:
                m = self._meets[idx] = _Meet(kind)
            elif m.kind != kind and m.error is None:
                m.error = CollectiveError(f"rank {rank} entered {kind!r} while others run {m.kind!r}")
                m.done = True
                self._cond.notify_all()
            m.payloads[rank] = payload
            if len(m.payloads) == self.size and not m.done:
                m.done = True
                self._cond.notify_all()
            deadline = time.monotonic() + timeout
            while not m.done:
                left = deadline - time.monotonic()
                if left <= 0:
                    m.error = CollectiveTimeout(kind, sorted(set(range(self.size)) - set(m.payloads)))
                    m.done = True
                    self._cond.notify_all()
                    break
                self._cond.wait(left)
            err, out = m.error, [m.payloads.get(r) for r in range(self.size)]
            m.taken += 1
            if m.taken == self.size:
                self._meets.pop(idx, None)
        if err is not None:
            raise err
        return out

    def run(self, fn, *args) -> list:
        """fn(rank, transport, *args) on every thread-rank, each on its own
        stream of the world's device; re-raise the first real failure ahead of
        the timeouts it caused (comm.py:262-284)."""
        results: list = [None] * self.size
        errors: list = [None] * self.size
        main = torch.cuda.current_stream(self.device)

        def body(r: int) -> None:
            try:
                torch.cuda.set_device(self.device)
                s = torch.cuda.Stream(device=self.device)
                s.wait_stream(main)
                with torch.cuda.stream(s):
                    results[r] = fn(r, self.transport(r), *args)
                _lib.host_wait(s)
            except BaseException as exc:  # noqa: BLE001
                errors[r] = exc

        threads = [threading.Thread(target=body, args=(r,), name=f"loopback-rank{r}") for r in range(self.size)]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        first = next((e for e in errors if e is not None and not isinstance(e, CollectiveTimeout)), None)
        first = first or next((e for e in errors if e is not None), None)
        if first is not None:
            raise first
        return results


def _ready_event() -> torch.cuda.Event:
    ev = torch.cuda.Event()
    ev.record()
    return ev


class LoopbackTransport:
    """TorchTransport's interface for thread-rank ``rank`` of a LoopbackWorld."""

    backend = "loopback"

    def __init__(self, world: LoopbackWorld, rank: int):
        self.world = world
        self.size = world.size
        self.rank = rank
        self.store = None

    def _exchange(self, kind: str, payload) -> list:
        """Meet with an event marking this rank's input ready; this rank's
        stream then waits for every peer's input."""
        got = self.world.meet(self.rank, kind, (payload, _ready_event()))
        cur = torch.cuda.current_stream()
        for _, ev in got:
            cur.wait_event(ev)
        return [p for p, _ in got]

    def _release(self, kind: str) -> None:
        """Peers' streams wait until this rank's copies are done (inputs stay
        valid until every reader has consumed them)."""
        got = self.world.meet(self.rank, kind + ":done", _ready_event())
        cur = torch.cuda.current_stream()
        for ev in got:
            cur.wait_event(ev)

    def all_gather_into_tensor(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        peers = self._exchange("all_gather", inp)
        n = inp.numel()
        for r, t in enumerate(peers):
            out[r * n:(r + 1) * n].copy_(t.reshape(-1))
        self._release("all_gather")

    def all_to_all_single(self, out: torch.Tensor, inp: torch.Tensor, out_splits: list[int],
                          in_splits: list[int]) -> None:
        peers = self._exchange("all_to_all", (inp, list(in_splits)))
        dst = 0
        for r, (t, splits) in enumerate(peers):
            off = sum(splits[: self.rank])
            cnt = splits[self.rank]
            if cnt != out_splits[r]:
                raise CollectiveError("all_to_all split sizes disagree across ranks")
            out[dst:dst + cnt].copy_(t[off:off + cnt])
            dst += cnt
        self._release("all_to_all")

    def all_reduce(self, t: torch.Tensor, op: str = "sum") -> None:
        peers = self._exchange("all_reduce", t.clone())
        acc = peers[0].clone()
        for x in peers[1:]:
            if op == "sum":
                acc += x
            elif op == "max":
                torch.maximum(acc, x, out=acc)
            else:
                torch.minimum(acc, x, out=acc)
        self._release("all_reduce")
        t.copy_(acc)

    def barrier(self) -> None:
        self._exchange("barrier", None)

    def peer_buffer(self, nbytes: int, device) -> PeerBuffer:
        ok = self.rank != self.world.fail_peer_rank
        local = torch.zeros(TV_PEER_HEADER + nbytes, dtype=torch.uint8, device=device) if ok else None
        _lib.host_wait()  # headers are zero before any peer posts
        everyone = self.world.meet(self.rank, "peer_buffer", local)
        if any(t is None for t in everyone):
            raise PeerMemoryUnavailable("peer memory: allocate failed on another rank"
                                        if ok else "peer memory: allocate failed (test hook)")
        return PeerBuffer(local, [t.data_ptr() for t in everyone], keep=everyone)

    def absent_ranks(self, rank: int, seq: int, issued: int, grace: float) -> list[int]:
        with self.world._cond:
            self.world.issued[rank] = issued
        deadline = time.monotonic() + grace
        while True:
            with self.world._cond:
                absent = [r for r in range(self.size) if r != rank and self.world.issued[r] < seq]
            if not absent or time.monotonic() >= deadline:
                return absent
            time.sleep(0.01)

    def check_kind(self, rank: int, seq: int, kind: str, timeout: float) -> tuple[list[int], dict]:
        try:
            got = self.world.meet(rank, "check", kind, timeout)
        except CollectiveTimeout as exc:
            return list(exc.absent), {rank: kind}
        return [], dict(enumerate(got))

    def abort(self) -> None:
        pass

    @staticmethod
    def is_timeout(exc: BaseException) -> bool:
        return isinstance(exc, CollectiveTimeout)
