"""Final log rows of the device loop at configs 1 and 2 (200 iterations, the
SURVEY 8d schedule) next to the reference's own rows (tests/golden)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_loop import _run  # noqa: E402

for name in ("cfg1_log.json", "cfg2_log.json"):
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", name)))
    rows, info, st, grid = _run(gold["spec"], gold["grid"], gold["max_iters"])
    got, ref = np.array(rows, float), np.array(gold["rows"])
    dev = np.abs(got[:, 1] - ref[:, 1]) / ref[:, 1]
    first_bad = int(np.argmax(dev > 1e-9)) if (dev > 1e-9).any() else None
    print(json.dumps({"golden": name, "final_gpu": list(map(float, got[-1])),
                      "final_ref": list(map(float, ref[-1])),
                      "max_rel_dev_first_150": float(dev[:151].max()),
                      "first_row_over_1e-9": first_bad}))
