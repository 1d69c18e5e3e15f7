"""Exchange microbenchmarks: the reference's `bench` sweep (`shufflecast/
bench.py:41-159`, driven by `cli.py bench`) on real NCCL collectives.

Every rank contributes one contiguous buffer of `msg` bytes per repetition
(`bench.py:86-116`):

* ``shuffle``       -- the buffer is cut N ways (`_split_points`) and slice d
  goes to rank d in one all-to-all-v (Alg. 1's data step);
* ``broadcast``     -- every rank is a root once: N broadcasts of `msg` bytes
  into an N*msg receive buffer in rank order (Alg. 2);
* ``broadcast_p2p`` -- each root's collective replaced by N-1 grouped sends.

Throughput = msg * N / 1e9 / elapsed (GB/s, `bench.py:141-143`, 1 GB = 1e9 B
as in `topology.py:20`), elapsed = mean over repetitions of the max over
ranks, each repetition bracketed by barriers.  On GPUs the repetition is
timed with CUDA events on the current stream; with gloo (CPU tests) by the
host clock.  Next to every measured row stands the paper's analytic model for
the same topology (`models.py:65-89`: shuffle k^2 B_g/(k-1) inside one
machine, broadcast k B_g/(k-1); multi-machine forms likewise), with
relative_error = |model - measured| / measured as in `bench.py:156-159` --
the reference prints this overlay only for its simulator, here it sits
beside real NVLink measurements.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

from .cluster import Endpoint, barrier

BENCH_OPS = ("shuffle", "broadcast", "broadcast_p2p")
DEFAULT_MESSAGE_CAP = 1 << 30
GB = 1e9
ROW_FIELDS = ["op", "msg_bytes", "k", "v", "bn_gbps", "bg_gbps", "efficiency",
              "measured_thpt_gbps", "model_thpt_gbps", "relative_error"]


class BenchError(ValueError):
    pass


def model_throughput(op: str, topo) -> float:
    """Paper model throughput in GB/s (models.py:65-89); broadcast_p2p is
    compared with the collective broadcast model (bench.py:114-119)."""
    import math
    k, v = topo.k, topo.v
    bg = topo.bg_gbps * (getattr(topo, "bg_efficiency", None) or topo.efficiency)
    bn = topo.bn_gbps * (getattr(topo, "bn_efficiency", None) or topo.efficiency)
    if k * v == 1:
        return math.inf
    if op == "shuffle":
        return k * k * bg / (k - 1) if v == 1 else (1.0 + 1.0 / (v - 1)) * v * bn
    if v == 1:
        return k * bg / (k - 1)
    return (1.0 + 1.0 / (v - 1)) * (k * bn * bg) / (k * bg + (k - 1) * bn)


@dataclass
class Topology:
    """The echoed topology columns (`topology.py` Topology: k GPUs per
    machine, v machines); k*v must equal the job's world size."""

    k: int
    v: int = 1
    bg_gbps: float = 450.0
    bn_gbps: float = 50.0
    efficiency: float = 0.8

    @property
    def n(self) -> int:
        return self.k * self.v


def parse_shorthand(label: str) -> tuple[int, int]:
    """'8x1' -> (8, 1) (`topology.py` parse_shorthand)."""
    try:
        k, v = (int(x) for x in label.lower().split("x"))
    except ValueError:
        raise BenchError(f"topology label {label!r} is not KxV") from None
    if k < 1 or v < 1:
        raise BenchError(f"topology label {label!r} needs K, V >= 1")
    return k, v


@dataclass
class BenchSpec:
    """One sweep: an exchange op over strictly increasing message sizes
    (`bench.py:50-76`, same validation and messages)."""

    op: str
    message_bytes: list[int]
    topology: Topology
    repetitions: int = 1
    max_message_bytes: int = DEFAULT_MESSAGE_CAP

    def __post_init__(self) -> None:
        if self.op not in BENCH_OPS:
            raise BenchError(f"unknown bench op {self.op!r}; choose from {BENCH_OPS}")
        if self.repetitions < 1:
            raise BenchError("repetitions must be >= 1")
        if not self.message_bytes:
            raise BenchError("empty message size sweep")
        if any(b <= 0 for b in self.message_bytes):
            raise BenchError("message sizes must be positive")
        if any(b >= a for b, a in zip(self.message_bytes, self.message_bytes[1:])):
            raise BenchError("message size sweep must be strictly increasing")
        over = [b for b in self.message_bytes if b > self.max_message_bytes]
        if over:
            raise BenchError(f"sweep sizes {over} exceed the configured memory cap "
                             f"of {self.max_message_bytes} bytes")


def _split_points(total: int, parts: int) -> list[int]:
    return [total * i // parts for i in range(parts + 1)]


def _step(ep: Endpoint, op: str, buf, out) -> None:
    """One repetition: every rank contributes `buf` (`bench.py:86-116`)."""
    import torch.distributed as dist
    from .exchange import alltoallv
    n, msg = ep.n, buf.numel()
    if op == "shuffle":
        cuts = _split_points(msg, n)
        send = [cuts[d + 1] - cuts[d] for d in range(n)]
        recv = [cuts[ep.rank + 1] - cuts[ep.rank]] * n
        alltoallv(ep, buf, send, recv)
        return
    out[ep.rank * msg:(ep.rank + 1) * msg].copy_(buf)
    if n == 1:
        return
    if op == "broadcast":
        for root in range(n):
            seg = out[root * msg:(root + 1) * msg]
            dist.broadcast(seg, src=root, group=ep.group)
        return
    ops = []
    for peer in range(n):
        if peer != ep.rank:
            ops.append(dist.P2POp(dist.isend, buf, peer, group=ep.group))
            ops.append(dist.P2POp(dist.irecv, out[peer * msg:(peer + 1) * msg], peer,
                                  group=ep.group))
    for r in dist.batch_isend_irecv(ops):
        r.wait()


def _max_over_ranks(ep: Endpoint, x: float) -> float:
    if ep.n == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=ep.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=ep.group)
    return float(t.item())


def run_bench(ep: Endpoint, spec: BenchSpec) -> list[dict]:
    """Run the sweep on this job; one row per message size, identical on
    every rank (`bench.py:122-159`)."""
    import torch
    topo = spec.topology
    if topo.n != ep.n:
        raise BenchError(f"topology {topo.k}x{topo.v} has {topo.n} GPUs, the job has {ep.n}")
    dev = ep.device
    on_gpu = dev.type == "cuda"
    rows = []
    for msg in spec.message_bytes:
        buf = torch.full((msg,), ep.rank % 251 + 1, dtype=torch.uint8, device=dev)
        out = None if spec.op == "shuffle" else torch.empty(msg * ep.n, dtype=torch.uint8,
                                                            device=dev)
        _step(ep, spec.op, buf, out)           # warm-up: communicator + buffers
        elapsed = 0.0
        for _ in range(spec.repetitions):
            barrier(ep)
            if on_gpu:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _step(ep, spec.op, buf, out)
                e1.record()
                barrier(ep)
                dt = e0.elapsed_time(e1) / 1e3
            else:
                t0 = time.perf_counter()
                _step(ep, spec.op, buf, out)
                barrier(ep)
                dt = time.perf_counter() - t0
            elapsed += _max_over_ranks(ep, dt)
        elapsed /= spec.repetitions
        measured = msg * ep.n / GB / elapsed if elapsed > 0 else float("inf")
        model = model_throughput(spec.op, topo)
        finite = model != float("inf") and measured not in (0.0, float("inf"))
        rows.append({
            "op": spec.op, "msg_bytes": msg, "k": topo.k, "v": topo.v,
            "bn_gbps": topo.bn_gbps, "bg_gbps": topo.bg_gbps, "efficiency": topo.efficiency,
            "measured_thpt_gbps": measured,
            "model_thpt_gbps": model if finite else None,
            "relative_error": abs(model - measured) / measured if finite else None,
        })
        del buf, out
    return rows
