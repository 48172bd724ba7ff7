"""Golden outputs of the reference's bench report helpers (deskrl bench.py:72-83,
221-236, 254-296), for paper_2502_08844_b200.stagebench.

    python tests/golden/make_golden_stagebench.py     (needs /root/reference; CPU)

Bootstrap CIs of fixed rate samples, the amortized breakdown of the published
timings, and the CSV + text table report_emit writes for a fixed report.
"""
import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from deskrl import bench

    rng = np.random.default_rng(3)
    samples = [list(rng.uniform(1e5, 2e5, k)) for k in (1, 2, 5, 20)]
    cis = [list(bench._bootstrap_ci(s, np.random.default_rng(1))) for s in samples]
    brk = {k: list(bench.amortized_breakdown(*v).fractions)
           for k, v in bench.PUBLISHED_TIMINGS.items()}
    rep = bench.ThroughputReport()
    rows = [("EnvStep", 1024, 0, 20, 123456.789, 120000.5, 130000.25, False),
            ("WithPixels", 256, 64, 20, 3400.125, 3300.0, 3500.0, False),
            ("WithInference", 256, 64, 1, 2900.0, 2900.0, 2900.0, True)]
    for r in rows:
        rep.results.append(bench.StageResult(*r))
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "bench.csv")
        table = bench.report_emit(rep, p)
        csv_text = open(p).read()
    data = {"samples": samples, "cis": cis, "breakdown": brk, "rows": rows, "csv": csv_text,
            "table": table}
    path = os.path.join(OUT, "stagebench_golden.json")
    with open(path, "w") as f:
        json.dump(data, f, indent=1)
    print(f"wrote {path}")


if __name__ == "__main__":
    main()
