"""Write tests/golden/gen_digests.json: SHA-256 of seconds 0..2 of each (family, traffic).

Calls only lmsgen (the shared input generator).  Re-run only when the generator
recipe (SURVEY.md Appendix A / DESIGN.md §4) is deliberately changed.
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import lmsgen as g  # noqa: E402

CASES = ["LR:B(1)", "LR:U(2.5)", "LR:R(0.1,5)", "CM:B(1)", "CM:U(2.5)", "CM:R(0.1,5)"]


def main():
    out = {"seed": g.SEED, "seconds": [0, 1, 2], "digests": {}}
    for key in CASES:
        fam, traffic = key.split(":")
        h = hashlib.sha256()
        for _, data in g.stream_datasets(fam, traffic, 3):
            h.update(data)
        out["digests"][key] = h.hexdigest()
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gen_digests.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
        fh.write("\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
