"""The JSON-lines server against the reference's own session
(tests/golden/serve_session.jsonl, produced by deskrl.serve.serve_stdio).

Same replies op by op: errors verbatim; observations / rewards within the
float64 env tolerance (1e-9 relative, floor 1e-3); flags exact; pixels
bit-exact up to edge pixels.  One documented deviation: the reference's
make_env fails with an internal error on a fresh env (Environment.
observation_shapes reads self.state before the first reset, envkit.py:579-584)
after registering the handle; ours returns the documented handle + shapes."""
import io
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_serve_session_matches_reference():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_08844_b200 import serve
    from tests.conftest import GOLDEN

    pairs = [json.loads(l) for l in open(os.path.join(GOLDEN, "serve_session.jsonl"))]
    reqs = [p["request"] for p in pairs]
    out = io.StringIO()
    serve.serve_stdio(io.StringIO("\n".join(json.dumps(r) for r in reqs) + "\n"), out)
    mine = [json.loads(l) for l in out.getvalue().strip().split("\n")]
    assert len(mine) == len(pairs)
    handle = 0
    for p, got in zip(pairs, mine):
        want, req = p["reply"], p["request"]
        if req["op"] == "make_env" and not want["ok"] and want["error"].startswith("internal"):
            handle += 1
            assert got["ok"] and got["handle"] == handle, got
            assert got["num_envs"] == req["config"].get("num_envs", 1)
            continue
        assert got["ok"] == want["ok"], (req, got, want)
        if not want["ok"]:
            assert got["error"] == want["error"]
            continue
        if "observation" in want:
            assert set(got["observation"]) == set(want["observation"])
            for k, v in want["observation"].items():
                g = got["observation"][k]
                assert g["shape"] == v["shape"]
                a, b = np.array(g["data"]), np.array(v["data"])
                if k == "pixels":
                    assert np.count_nonzero(a != b) <= max(2, b.size // 10000)
                else:
                    assert np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-3)) <= 1e-9
        if "reward" in want:
            a, b = np.array(got["reward"]), np.array(want["reward"])
            assert np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-3)) <= 1e-9
            assert got["done"] == want["done"] and got["truncated"] == want["truncated"]
        for k in ("version",):
            if k in want:
                assert got[k] == want[k]
