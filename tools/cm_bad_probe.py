"""Diagnostics: run CM1S and CM2S over the same freshly generated 10M-record batches several
times and print each batch's bad / record counts (a valid generator stream has none bad)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_04289_b200 as P  # noqa: E402
from paper_2111_04289_b200 import _lib as L  # noqa: E402
from lmsgen import cuda as gcu  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
for rep in range(3):
    bufs = [gcu.second_tensor("CM", t, n) for t in range(3)]
    for kind in ("CM1S", "CM2S", "CM1S"):
        q = P.Query(kind, mode="manual", max_batch_bytes=1 << 20, max_result_rows=1 << 22)
        out = []
        for t, (b, nb) in enumerate(bufs):
            q.push_device(b.data_ptr(), nb, float(t))
            q.force(t + 1.0)
            q.sync(ok=(L.LMS_OK, L.LMS_EFORMAT))
            r = q.record(t)
            out.append((r["num_records"], r["bad_records"]))
        q.close()
        print(rep, kind, out, flush=True)
    # byte-level check of the generated data: every line has 12 commas
    for t, (b, nb) in enumerate(bufs):
        x = b[:nb]
        nl = (x == 10).sum().item()
        cm = (x == 44).sum().item()
        print(f"  data t={t}: {nb} B, newlines {nl}, commas {cm} (12 per line: {cm == 12 * nl})", flush=True)
