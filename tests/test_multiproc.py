"""N > 1 host protocol on CPU: world-size-2 (and 3) gloo process groups.

Only one GPU is available to this build, so the multi-rank exchange path is
exercised here with gloo and CPU tensors: size exchange, the shuffle's
all-to-all-v receive order (source rank ascending, input order within a
rank, exchange.py:52-56,161-166), broadcast (Alg. 2 and p2p) concatenation
in rank order (exchange.py:274-276), the final gather to rank 0
(engine.py:345-365), column-range metadata merging and the schema
rendezvous error.  The on-device partition kernels are replaced by the CPU
oracle's hash_partition inside the children (it is checked against the
kernel separately in test_gpu_parity.py).
"""

import os
import socket
import traceback

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cpu_table(rank: int, n: int, seed: int):
    from paper_2506_09226_b200.table import Column, ColumnTable
    rng = np.random.default_rng(seed + rank)
    k = rng.integers(0, 50, size=n).astype(np.int64)
    v = (np.arange(n) + 1000 * rank).astype(np.int32)
    d = rng.integers(0, 3, size=n).astype(np.uint8)
    return ColumnTable({
        "k": Column("int64", torch.from_numpy(k), 0, None, int(k.min(initial=0)), int(k.max(initial=-1))),
        "v": Column("int64", torch.from_numpy(v), 0, None, int(v.min(initial=0)), int(v.max(initial=-1))),
        "d": Column("dict", torch.from_numpy(d), 0, ("x", "y", "z"), 0, 2),
    })


def _as_oracle(t):
    return {n: (c.kind, c.data.numpy().astype(np.int64), c.dictionary) for n, c in t.columns.items()}


class _HostPartitioner:
    """CPU stand-in for exchange._Partitioner (same contract: counts after
    pass 1, local() = every column partitioned in bucket order)."""

    def __init__(self, table, key_columns, n_parts):
        from oracle import ref as O
        from paper_2506_09226_b200.exchange import _key_cols
        self.table = table.materialize()
        _key_cols(self.table, key_columns)
        self.names = self.table.column_names
        self.n = self.table.row_count
        self.n_parts = n_parts
        b = O.hash_keys(_as_oracle(self.table), key_columns) % np.uint64(n_parts)
        self.order = torch.from_numpy(np.argsort(b, kind="stable"))
        self.counts = np.bincount(b.astype(np.int64), minlength=n_parts).astype(np.int64)

    def local(self, cols):
        return [cols[nm].data[self.order] for nm in self.names]


def _worker(rank, world, port, seed, out_q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                          WORLD_SIZE=str(world))
        import paper_2506_09226_b200 as P
        from paper_2506_09226_b200 import exchange as X
        from paper_2506_09226_b200.engine import DeviceContext
        from paper_2506_09226_b200.table import SchemaError
        import torch.distributed as dist
        X._Partitioner = _HostPartitioner
        ep = P.create_cluster("gloo")
        res = {"rank": ep.rank, "n": ep.n}
        t = _cpu_table(rank, 40 + 7 * rank, seed)
        # size exchange: column `rank` of the N x N matrix
        row = np.asarray([10 * rank + j for j in range(world)], dtype=np.int64)
        inc, offs = P.size_exchange(ep, row)
        res["incoming"] = inc.tolist()
        res["offsets"] = offs.tolist()
        st = P.ExchangeStats()
        sh = P.shuffle_table(ep, t, ["k"], st)
        res["shuffle"] = {n: c.data.numpy().tolist() for n, c in sh.columns.items()}
        res["shuffle_range"] = (sh.column("k").lo, sh.column("k").hi)
        res["shuffle_msgs"] = st.messages
        for p2p in (False, True):
            bc = P.broadcast_table(ep, t, None, use_p2p=p2p)
            res[f"bcast_{p2p}"] = {n: c.data.numpy().tolist() for n, c in bc.columns.items()}
        ctx = DeviceContext(ep, {}, timed=False)
        g = ctx.gather(t)
        res["gather"] = None if g is None else {n: c.data.numpy().tolist()
                                                for n, c in g.columns.items()}
        # a schema mismatch is detected on every rank
        bad = t if rank == 0 else t.select(["k", "v"])
        try:
            P.shuffle_table(ep, bad, ["k"])
            res["schema_error"] = False
        except SchemaError:
            res["schema_error"] = True
        res["all_gather"] = X.all_gather_tensor(ep, torch.tensor([rank, 7 * rank])).tolist()
        dist.barrier()
        dist.destroy_process_group()
        out_q.put(res)
    except Exception:  # pragma: no cover - surfaced in the parent
        out_q.put({"rank": rank, "error": traceback.format_exc()})


def _run(world: int, seed: int = 3):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r = q.get(timeout=240)
        assert "error" not in r, r["error"]
        out[r["rank"]] = r
    for p in procs:
        p.join(timeout=60)
    return out


@pytest.fixture(scope="module", params=[2, 3])
def world(request):
    return request.param, _run(request.param)


def test_size_exchange_matrix_column(world):
    n, res = world
    for r in range(n):
        assert res[r]["incoming"] == [10 * s + r for s in range(n)]
        assert res[r]["offsets"] == list(np.cumsum([0] + res[r]["incoming"][:-1]))


def test_shuffle_matches_reference_semantics(world):
    """rank j holds hash_partition(src)[j] for every src, in source-rank order."""
    from oracle import ref as O
    n, res = world
    parts = [O.hash_partition(_as_oracle(_cpu_table(r, 40 + 7 * r, 3)), ["k"], n)
             for r in range(n)]
    total = 0
    for j in range(n):
        exp = {c: np.concatenate([parts[s][j][c][1] for s in range(n)]).tolist()
               for c in ("k", "v", "d")}
        assert res[j]["shuffle"] == exp
        total += len(exp["k"])
        ks = exp["k"]
        if ks:
            lo, hi = res[j]["shuffle_range"]
            assert lo <= min(ks) and max(ks) <= hi
    assert total == sum(40 + 7 * r for r in range(n))          # conservation


def test_broadcast_is_rank_ordered_concat(world):
    n, res = world
    exp = {c: np.concatenate([_as_oracle(_cpu_table(r, 40 + 7 * r, 3))[c][1]
                              for r in range(n)]).tolist() for c in ("k", "v", "d")}
    for r in range(n):
        assert res[r]["bcast_False"] == exp
        assert res[r]["bcast_True"] == exp


def test_gather_to_root(world):
    n, res = world
    exp = {c: np.concatenate([_as_oracle(_cpu_table(r, 40 + 7 * r, 3))[c][1]
                              for r in range(n)]).tolist() for c in ("k", "v", "d")}
    assert res[0]["gather"] == exp
    assert all(res[r]["gather"] is None for r in range(1, n))


def test_schema_mismatch_and_all_gather(world):
    n, res = world
    assert all(res[r]["schema_error"] for r in range(n))
    assert all(res[r]["all_gather"] == [[s, 7 * s] for s in range(n)] for r in range(n))
