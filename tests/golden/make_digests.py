"""Reference result digests (engine.py:182-197 result_digest of
reference_run, engine.py:463-469) for the six reference queries, plus the
digest payload lines they hash, made by running the REAL reference in the
dev container.

    python tests/golden/make_digests.py   -> tests/golden/digests.json

The payload lines let a test tell a real mismatch from a rounding tie: the
digest prints floats at 10 significant digits, and where the exact decimal
sits on a tie at that digit (e.g. Q1 sum_disc_price 332048914.55) the
reference's float64 accumulation and the exact fixed-point value print
different last digits.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")


def payload(table):
    lines = []
    decoded = [table.column(n).decoded() for n in table.column_names]
    kinds = [table.column(n).kind for n in table.column_names]
    for i in range(table.row_count):
        lines.append("|".join(f"{col[i]:.9e}" if k == "float64" else str(col[i])
                              for col, k in zip(decoded, kinds)))
    lines.sort()
    return [",".join(table.column_names)] + lines


def main():
    import shufflecast as s
    out = {}
    for sf in (0.01, 0.1):
        ds = s.generate(sf, skew=0.0, seed=0)
        res = {q: s.reference_run(q, ds) for q in s.SUPPORTED_QUERIES}
        out[f"sf{sf}"] = {q: s.result_digest(r) for q, r in res.items()}
        out[f"lines_sf{sf}"] = {q: payload(r) for q, r in res.items()}
    with open(os.path.join(HERE, "digests.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print({k: v for k, v in out.items() if not k.startswith("lines")})


if __name__ == "__main__":
    main()
