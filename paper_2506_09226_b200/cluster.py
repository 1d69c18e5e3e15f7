"""Workers and their transports.

Mirrors the reference's transport layer
(`/root/reference/pkg/src/shufflecast/transport.py:32-442`) for the two ways
this package runs N workers:

* ``MODE_IN_PROCESS`` -- the reference's own mode: ``create_cluster(topo,
  MODE_IN_PROCESS)`` makes N endpoints in one process and ``run_workers``
  runs one thread per endpoint (transport.py:398-442).  Here every worker is a
  *virtual rank* on the current GPU: its tables live in that GPU's HBM, its
  kernels run on the device, and exchanges move device memory between the
  workers' buffers (the shuffle's partition kernel writes straight into the
  receivers' buffers, exchange.py).  All workers enqueue on the same CUDA
  stream, so stream order is the happens-before between a sender's writes
  and a receiver's reads; the rendezvous below only orders the host side.
  This runs every N>1 plan (shuffles, broadcasts, gathers, cross-rank folds)
  with real kernels on one B200.
* ``MODE_NCCL`` / ``MODE_GLOO`` -- one process per GPU (torchrun), the
  production layout: ``create_cluster()`` joins the job described by the
  RANK / WORLD_SIZE environment and returns this process's ``Endpoint``.

The reference's virtual-time simulator (``MODE_SIMULATED``,
transport.py:300-339) is out of scope: device time replaces
it.  Errors keep the reference's types: ``ClusterConfigError``,
``ProtocolError``, ``DeadlockError`` (transport.py:36-53).
"""

from __future__ import annotations

import os
import threading
from collections import deque
from dataclasses import dataclass, field

MODE_NCCL = "nccl"
MODE_GLOO = "gloo"
MODE_IN_PROCESS = "in_process"
MODE_SIMULATED = "simulated"
DEFAULT_EFFICIENCY = 0.8


class TransportError(RuntimeError):
    pass


class ClusterConfigError(TransportError):
    """Ranks or cluster shapes that do not exist."""


class ProtocolError(TransportError):
    """Workers disagree about a collective operation."""


class DeadlockError(TransportError):
    """A collective could not be matched across ranks."""


class _Aborted(TransportError):
    """A peer failed; this worker unwinds quietly (transport.py:52)."""


class TopologyError(ValueError):
    """Invalid cluster shape or bandwidth (topology.py:27)."""


@dataclass(frozen=True)
class Topology:
    """``v`` machines with ``k`` GPUs each (topology.py:31-60).  Only the
    shape is used here; the bandwidth fields feed the analytic models, which
    are out of scope."""

    k: int
    v: int
    bg_gbps: float = 900.0
    bn_gbps: float = 900.0
    efficiency: float = DEFAULT_EFFICIENCY
    bg_efficiency: float | None = None
    bn_efficiency: float | None = None

    def __post_init__(self) -> None:
        if self.k < 1:
            raise TopologyError(f"k must be >= 1, got {self.k}")
        if self.v < 1:
            raise TopologyError(f"V must be >= 1, got {self.v}")
        if self.bg_gbps <= 0 or self.bn_gbps <= 0:
            raise TopologyError(f"bandwidths must be positive, got bg={self.bg_gbps} "
                                f"bn={self.bn_gbps}")
        for name, eff in (("efficiency", self.efficiency), ("bg_efficiency", self.bg_efficiency),
                          ("bn_efficiency", self.bn_efficiency)):
            if eff is not None and not 0.0 < eff <= 1.0:
                raise TopologyError(f"{name} must be in (0, 1], got {eff}")

    @property
    def n(self) -> int:
        return self.k * self.v

    def node_of(self, rank: int) -> int:
        return rank // self.k

    def local_index_of(self, rank: int) -> int:
        return rank % self.k


@dataclass
class GroupOp:
    """One entry of a grouped communication step (transport.py:94-110).

    kind "send": ``peer`` = destination, ``payload`` bytes-like / array /
    tensor; "recv": ``peer`` = source, ``nbytes`` = expected length;
    "bcast": ``peer`` = root, the root supplies ``payload``, the others an
    ``nbytes`` reservation.
    """

    kind: str
    peer: int
    payload: object | None = None
    nbytes: int | None = None
    tag: int = 0


@dataclass
class Endpoint:
    """A worker's handle (transport.py:126-167).  ``cluster`` is the
    in-process hub for ``MODE_IN_PROCESS`` and None for one-process-per-GPU
    jobs (``group`` is then the torch.distributed process group, None =
    WORLD).  Owned by one thread; not reentrant."""

    rank: int
    n: int
    backend: str
    group: object = None
    cluster: "Cluster | None" = field(default=None, repr=False)

    @property
    def in_process(self) -> bool:
        return self.cluster is not None

    @property
    def device(self):
        import torch
        if self.backend in (MODE_NCCL, MODE_IN_PROCESS):
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    @property
    def distributed(self) -> bool:
        return self.n > 1

    @property
    def node(self) -> int:
        return self.cluster.topology.node_of(self.rank) if self.cluster else 0

    @property
    def local_index(self) -> int:
        return self.cluster.topology.local_index_of(self.rank) if self.cluster else self.rank

    def send(self, dst: int, payload, tag: int = 0) -> None:
        """Point-to-point send (transport.py:154); in-process only."""
        self._hub("send")._send(self.rank, dst, payload, tag)

    def recv(self, src: int, tag: int = 0):
        """Blocking point-to-point receive (transport.py:157)."""
        return self._hub("recv")._recv(self.rank, src, tag)

    def _hub(self, what: str) -> "Cluster":
        if self.cluster is None:
            raise ClusterConfigError(f"{what}: point-to-point messages need an in-process cluster")
        return self.cluster


class _Rendezvous:
    __slots__ = ("slots", "labels", "done", "result", "error", "consumed")

    def __init__(self, n: int):
        self.slots: list = [None] * n
        self.labels: list = [None] * n
        self.done = False
        self.result = None
        self.error: BaseException | None = None
        self.consumed = 0


class Cluster:
    """Shared state of N in-process workers: mailboxes and the deterministic
    all-ranks rendezvous (transport.py:182-390)."""

    def __init__(self, topology: Topology, mode: str = MODE_IN_PROCESS, seed: int = 0):
        if mode == MODE_SIMULATED:
            raise ClusterConfigError("the virtual-time simulator (MODE_SIMULATED) is out of scope; "
                                     "use MODE_IN_PROCESS (device time is measured instead)")
        if mode != MODE_IN_PROCESS:
            raise ClusterConfigError(f"unknown transport mode {mode!r}")
        if topology.n < 1:
            raise ClusterConfigError("cluster needs at least one endpoint")
        self.topology = topology
        self.mode = mode
        self.seed = seed
        self.endpoints = [Endpoint(r, topology.n, MODE_IN_PROCESS, None, self)
                          for r in range(topology.n)]
        self._cond = threading.Condition(threading.RLock())
        self._mailboxes: dict[tuple[int, int, int], deque] = {}
        self._rendezvous: list = []
        self._next_step = [0] * topology.n
        self._waiting: dict[int, str] = {}
        self._finished: set[int] = set()
        self._abort: BaseException | None = None

    @property
    def n(self) -> int:
        return self.topology.n

    def _check_rank(self, rank: int, what: str) -> None:
        if not 0 <= rank < self.n:
            raise ClusterConfigError(f"{what} rank {rank} outside [0, {self.n})")

    # -- point-to-point ----------------------------------------------------
    def _send(self, src: int, dst: int, payload, tag: int) -> None:
        self._check_rank(dst, "destination")
        with self._cond:
            self._raise_if_broken()
            self._mailboxes.setdefault((src, dst, tag), deque()).append(payload)
            self._cond.notify_all()

    def _recv(self, rank: int, src: int, tag: int):
        self._check_rank(src, "source")
        key = (src, rank, tag)
        with self._cond:
            while True:
                self._raise_if_broken()
                box = self._mailboxes.get(key)
                if box:
                    return box.popleft()
                self._wait(rank, f"recv(src={src}, tag={tag})",
                           lambda: bool(self._mailboxes.get(key)))

    # -- rendezvous --------------------------------------------------------
    def rendezvous(self, rank: int, label: str, slot, commit):
        """Every worker calls in the same program order; the last arrival runs
        ``commit(slots)`` (slots in rank order) once and all get its result.
        Differing labels raise ProtocolError (transport.py:242-287)."""
        with self._cond:
            self._raise_if_broken()
            step = self._next_step[rank]
            self._next_step[rank] += 1
            while len(self._rendezvous) <= step:
                self._rendezvous.append(_Rendezvous(self.n))
            rdv = self._rendezvous[step]
            rdv.slots[rank] = slot
            rdv.labels[rank] = label
            if sum(1 for lb in rdv.labels if lb is not None) == self.n:
                labels = {lb for lb in rdv.labels}
                try:
                    if len(labels) > 1:
                        raise ProtocolError(f"collective mismatch at step {step}: workers "
                                            f"posted {sorted(labels)}")
                    rdv.result = commit(rdv.slots)
                except BaseException as exc:   # propagated to every participant
                    rdv.error = exc
                rdv.done = True
                self._cond.notify_all()
            else:
                while not rdv.done:
                    self._raise_if_broken()
                    self._wait(rank, f"collective {label!r} at step {step}", lambda: rdv.done)
            rdv.consumed += 1
            if rdv.consumed == self.n:
                self._rendezvous[step] = None  # release payload references
            if rdv.error is not None:
                raise rdv.error
            return rdv.result

    def _wait(self, rank: int, why: str, satisfiable) -> None:
        """Wait on the condition; every live worker blocked with nothing able
        to make progress is a deadlock (transport.py:351-371)."""
        self._waiting[rank] = (why, satisfiable)
        try:
            while not satisfiable():
                self._raise_if_broken()
                live = self.n - len(self._finished)
                # a waiter whose condition already holds has merely not woken
                # up yet: it is not blocked
                if (len(self._waiting) >= live
                        and not any(ok() for _, ok in self._waiting.values())):
                    desc = "; ".join(f"rank {r}: {w}" for r, (w, _) in sorted(self._waiting.items()))
                    raise DeadlockError(f"all live workers are blocked: {desc}")
                self._cond.wait(timeout=1.0)
        finally:
            self._waiting.pop(rank, None)

    def _raise_if_broken(self) -> None:
        if self._abort is not None:
            raise _Aborted(f"aborted by a peer failure: {self._abort!r}")

    def mark_finished(self, rank: int) -> None:
        with self._cond:
            self._finished.add(rank)
            self._cond.notify_all()

    def abort(self, exc: BaseException) -> None:
        with self._cond:
            if self._abort is None:
                self._abort = exc
            self._cond.notify_all()

    def reset(self) -> None:
        """Clear per-run state (run_workers calls it before starting)."""
        with self._cond:
            self._finished.clear()
            self._waiting.clear()
            self._abort = None
            self._rendezvous = []
            self._next_step = [0] * self.n
            self._mailboxes.clear()


def _dist_endpoint(backend: str | None) -> Endpoint:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if backend is None:
        backend = MODE_NCCL if torch.cuda.is_available() else MODE_GLOO
    if backend not in (MODE_NCCL, MODE_GLOO):
        raise ClusterConfigError(f"unknown backend {backend!r}")
    if world > 1 or dist.is_initialized():
        if backend == MODE_NCCL:
            local = int(os.environ.get("LOCAL_RANK", rank))
            torch.cuda.set_device(local)
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            kw = {}
            if backend == MODE_NCCL:
                kw["device_id"] = torch.device("cuda", torch.cuda.current_device())
            dist.init_process_group(backend, rank=rank, world_size=world, **kw)
        return Endpoint(dist.get_rank(), dist.get_world_size(), backend, None)
    if rank != 0:
        raise ClusterConfigError(f"rank {rank} outside a 1-rank job")
    return Endpoint(0, 1, backend, None)


def create_cluster(topo=None, mode: str | None = None, seed: int = 0):
    """``create_cluster(topo, MODE_IN_PROCESS, seed)`` -> in-process
    ``Cluster`` of ``topo.n`` virtual workers on this GPU
    (transport.py:398-400; ``topo`` may also be a worker count).

    ``create_cluster()`` / ``create_cluster("nccl" | "gloo")`` -> this
    process's ``Endpoint`` in the torchrun job (one process per GPU); a
    1-rank job when no torchrun environment is present.
    """
    if isinstance(topo, str) and mode is None:
        return _dist_endpoint(topo)
    if topo is None:
        return _dist_endpoint(mode)
    if isinstance(topo, int):
        topo = Topology(k=topo, v=1)
    if not isinstance(topo, Topology):
        raise ClusterConfigError(f"create_cluster: expected a Topology, got {type(topo).__name__}")
    return Cluster(topo, mode or MODE_IN_PROCESS, seed)


def run_workers(cluster, fn, *args) -> list:
    """Run ``fn(endpoint, *args)`` once per endpoint, one thread each; the
    per-rank results in rank order (transport.py:403-442).  A failing worker
    aborts its peers and its exception is re-raised (deadlocks reported only
    if nothing else failed).  For a process-per-GPU ``Endpoint`` this runs
    ``fn`` on the local rank and returns ``[result]``."""
    if isinstance(cluster, Endpoint):
        return [fn(cluster, *args)]
    cluster.reset()
    results: list = [None] * cluster.n
    failures: list[tuple[int, BaseException]] = []
    lock = threading.Lock()
    device = None
    try:
        import torch
        if torch.cuda.is_available():
            device = torch.cuda.current_device()
    except ImportError:  # pragma: no cover
        pass

    def body(ep: Endpoint) -> None:
        try:
            if device is not None:        # workers run on the caller's GPU
                import torch
                torch.cuda.set_device(device)
            results[ep.rank] = fn(ep, *args)
        except _Aborted:
            pass
        except BaseException as exc:      # noqa: BLE001 -- re-raised below
            with lock:
                failures.append((ep.rank, exc))
            cluster.abort(exc)
        finally:
            cluster.mark_finished(ep.rank)

    if cluster.n == 1:
        body(cluster.endpoints[0])
    else:
        threads = [threading.Thread(target=body, args=(ep,), name=f"worker-{ep.rank}")
                   for ep in cluster.endpoints]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    if failures:
        primary = [f for f in failures if not isinstance(f[1], DeadlockError)]
        raise (primary or failures)[0][1]
    return results


def barrier(ep: Endpoint) -> None:
    """All workers meet (collectives.py:216-223).  Process-per-GPU: the
    current stream is drained first.  In-process: host rendezvous only --
    the workers share one stream, so device order already follows issue
    order."""
    import torch
    if ep.in_process:
        if ep.n > 1:
            ep.cluster.rendezvous(ep.rank, "barrier", None, lambda _s: None)
        return
    if ep.backend == MODE_NCCL and torch.cuda.is_available():
        torch.cuda.synchronize()
    if ep.n > 1:
        import torch.distributed as dist
        dist.barrier(group=ep.group)
