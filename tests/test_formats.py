"""DSKRLCK1 checkpoints interchangeable with the reference's (CPU):
tests/golden/ref_checkpoint.bin was written by deskrl.ppo.save_checkpoint."""
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN

torch = pytest.importorskip("torch")


def _nets():
    from paper_2502_08844_b200 import rollout as R

    return R.make_policy(5, 1, (8, 8)), R.make_value(5, (6,))


def test_load_reference_checkpoint_and_write_identical_bytes(tmp_path):
    from paper_2502_08844_b200 import checkpoint as C

    ref = np.load(os.path.join(GOLDEN, "ref_checkpoint.npz"))
    path = os.path.join(GOLDEN, "ref_checkpoint.bin")
    policy, value = _nets()
    header, pn, vn = C.load_checkpoint(path, policy, value, device="cpu")
    assert header["extra"] == {"env_steps": 1234, "note": "golden"}
    for k, v in policy.state_dict().items():
        np.testing.assert_array_equal(v.numpy(), ref[f"policy/{k}"])
    for k, v in value.state_dict().items():
        np.testing.assert_array_equal(v.numpy(), ref[f"value/{k}"])
    for n, key in ((pn, "pn"), (vn, "vn")):
        c, m, var = n.to_numpy()
        assert c == float(ref[f"{key}/count"])
        np.testing.assert_array_equal(m, ref[f"{key}/mean"])
        np.testing.assert_array_equal(var, ref[f"{key}/var"])
    out = tmp_path / "mine.bin"
    C.save_checkpoint(out, policy, value, str(ref["config_hash"]), header["extra"], pn, vn)
    assert out.read_bytes() == open(path, "rb").read()
    assert C.read_checkpoint_header(out)["config_hash"] == str(ref["config_hash"])
    with pytest.raises(C.ConfigError):
        C.load_checkpoint(path, policy, value, config_hash="0" * 16, device="cpu")
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTACKPT" + b"\0" * 16)
    with pytest.raises(C.ConfigError):
        C.read_checkpoint_header(bad)
