"""Stable compaction of 1/2/4/8-byte columns at selectivities from none to
all rows (the staged regions moved into place by the 16-byte-chunk
region copy: every destination alignment occurs), and result reads through
the mapped / copy paths of table.to_host -- against numpy."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 1000, 300_001, 2_500_003])
@pytest.mark.parametrize("frac", [0.0, 0.001, 0.37, 1.0])
def test_filter_materialize_all_widths(n, frac):
    from paper_2506_09226_b200.table import Column, ColumnTable
    import paper_2506_09226_b200 as P
    rng = np.random.default_rng(n + int(frac * 1000))
    sel = rng.integers(0, 1_000_000, size=n)
    cols = {
        "s": ("int64", sel),
        "u8": ("dict", rng.integers(0, 200, size=n)),                    # 1-byte codes
        "i16": ("date32", rng.integers(-20000, 20000, size=n)),
        "i32": ("int64", rng.integers(-2**30, 2**30, size=n)),
        "i64": ("int64", rng.integers(-2**62, 2**62, size=n)),
    }
    dicts = {"u8": tuple(f"v{i:03d}" for i in range(200))}
    t = ColumnTable({k: Column.from_numpy(kind, v, dicts.get(k)) for k, (kind, v) in cols.items()})
    cut = int(frac * 1_000_000)
    got = P.filter_table(t, t["s"] < cut).materialize()
    m = sel < cut
    for k, (_, v) in cols.items():
        assert np.array_equal(got.column(k).values, v[m]), (k, n, frac)


def test_to_host_paths(monkeypatch):
    import torch
    from paper_2506_09226_b200 import table as T
    for n in (0, 1, 3, 17, 4096, (1 << 20) // 8 + 5, 3 << 20):
        x = torch.arange(n, dtype=torch.int64, device="cuda") * 7 - 5
        assert np.array_equal(T.to_host(x), np.arange(n, dtype=np.int64) * 7 - 5)
    y = torch.arange(999, dtype=torch.int16, device="cuda")
    assert np.array_equal(T.to_host(y[1::2]), np.arange(999, dtype=np.int16)[1::2])
    monkeypatch.setattr(T, "_MAPPED_OK", False)
    assert np.array_equal(T.to_host(y), np.arange(999, dtype=np.int16))
