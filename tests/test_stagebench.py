"""Bench report schema: paper_2502_08844_b200.stagebench
against the reference's own bench helpers (tests/golden/stagebench_golden.json):
bootstrap CIs, amortized breakdown, CSV bytes and text table; plus the device
measure_stage rows on the GPU."""
import json
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLDEN, "stagebench_golden.json")) as f:
        return json.load(f)


def test_bootstrap_ci_matches_reference(gold):
    from paper_2502_08844_b200 import stagebench as sb

    for s, ci in zip(gold["samples"], gold["cis"]):
        assert list(sb._bootstrap_ci(s, np.random.default_rng(1))) == ci


def test_breakdown_matches_reference(gold):
    from paper_2502_08844_b200 import stagebench as sb

    timings = {"CartpoleBalance": (7.30e-7, 2.48e-6, 2.93e-6, 3.20e-5),
               "PandaPickCubeCartesian": (1.56e-5, 2.71e-5, 2.78e-5, 6.39e-5)}
    for k, v in timings.items():
        assert list(sb.amortized_breakdown(*v).fractions) == gold["breakdown"][k]
    with pytest.raises(sb.MeasurementAnomaly):
        sb.amortized_breakdown(2.0, 1.0, 3.0, 4.0)


def test_report_csv_and_table_byte_identical(gold, tmp_path):
    from paper_2502_08844_b200 import stagebench as sb

    rep = sb.ThroughputReport([sb.StageResult(*r) for r in gold["rows"]])
    p = tmp_path / "bench.csv"
    table = sb.report_emit(rep, p)
    assert p.read_text() == gold["csv"]
    assert table == gold["table"]
    rows = sb.report_parse(p)
    assert [r["stage"] for r in rows] == ["EnvStep", "WithPixels", "WithInference"]
    bad = tmp_path / "bad.csv"
    bad.write_text("stage,batch\nEnvStep,1\n")
    with pytest.raises(sb.ConfigError):
        sb.report_parse(bad)


@pytest.mark.gpu
def test_measure_stage_device(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_08844_b200 as dk
    from paper_2502_08844_b200 import stagebench as sb

    cfg = dk.EnvConfig(task="cartpole-balance-pixels")
    rep = sb.ThroughputReport()
    for st in (sb.Stage.ENV_STEP, sb.Stage.WITH_PIXELS, sb.Stage.WITH_INFERENCE):
        r = sb.measure_stage(st, cfg, num_envs=256, repetitions=5, steps_per_batch=4)
        assert r.median_sps > 0 and r.ci_low <= r.median_sps <= r.ci_high
        assert r.resolution == (0 if st == sb.Stage.ENV_STEP else 64)
        rep.results.append(r)
    t = [1.0 / r.median_sps for r in rep.results]
    assert t[0] < t[1] < t[2]  # physics < + render < + inference
    sb.report_emit(rep, tmp_path / "b.csv")
    assert len(sb.report_parse(tmp_path / "b.csv")) == 3
    r = sb.measure_stage(sb.Stage.WITH_INFERENCE, dk.EnvConfig(task="cartpole-balance"),
                         num_envs=256, repetitions=3, steps_per_batch=4)
    assert r.resolution == 0 and r.median_sps > 0
    with pytest.raises(dk.ConfigError):
        sb.measure_stage(sb.Stage.WITH_PIXELS, dk.EnvConfig(task="cartpole-balance"))
    with pytest.raises(dk.ConfigError):
        sb.measure_stage(sb.Stage.AND_TRAINING, cfg)
