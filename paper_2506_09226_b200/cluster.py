"""One process per GPU over torch.distributed (NCCL on B200, gloo on CPU).

Replaces the reference's thread-per-worker in-process transport
(`/root/reference/pkg/src/shufflecast/transport.py:126-442`): an
``Endpoint`` is this process's rank in the job; ``Cluster`` is the process
group.  The reference's rendezvous-based protocol checks become collective
shape checks that raise the same exception types (``ProtocolError``,
``DeadlockError``, ``ClusterConfigError``, transport.py:36-53).
The virtual-time simulator is out of scope: device time
replaces it.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

MODE_NCCL = "nccl"
MODE_GLOO = "gloo"


class TransportError(RuntimeError):
    pass


class ClusterConfigError(TransportError):
    """Ranks or cluster shapes that do not exist."""


class ProtocolError(TransportError):
    """Workers disagree about a collective operation."""


class DeadlockError(TransportError):
    """A collective could not be matched across ranks."""


@dataclass
class Endpoint:
    """This process's handle into the job (transport.py:126-167)."""

    rank: int
    n: int
    backend: str
    group: object = None

    @property
    def device(self):
        import torch
        if self.backend == MODE_NCCL:
            return torch.device("cuda", torch.cuda.current_device())
        return torch.device("cpu")

    @property
    def distributed(self) -> bool:
        return self.n > 1


def create_cluster(backend: str | None = None) -> Endpoint:
    """Join the job described by torchrun env vars (RANK/WORLD_SIZE/...).

    Without them this is a single-rank cluster and no process group is made.
    """
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


def barrier(ep: Endpoint) -> None:
    """All ranks meet; on GPUs the current stream is drained first
    (collectives.py:216-223)."""
    import torch
    if ep.backend == MODE_NCCL and torch.cuda.is_available():
        torch.cuda.synchronize()
    if ep.n > 1:
        import torch.distributed as dist
        dist.barrier(group=ep.group)
