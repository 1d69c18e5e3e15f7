"""Reference result digests (engine.py:182-197 result_digest of
reference_run, engine.py:463-469) for the six reference queries, made by
running the REAL reference in the dev container.

    python tests/golden/make_digests.py   -> tests/golden/digests.json
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")


def main():
    import shufflecast as s
    out = {}
    for sf in (0.01, 0.1):
        ds = s.generate(sf, skew=0.0, seed=0)
        out[f"sf{sf}"] = {q: s.result_digest(s.reference_run(q, ds)) for q in s.SUPPORTED_QUERIES}
    with open(os.path.join(HERE, "digests.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(out)


if __name__ == "__main__":
    main()
