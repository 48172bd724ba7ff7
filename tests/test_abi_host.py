"""CPU-side checks: the C-ABI library loads and exports every symbol declared
in include/deskrl_b200.h; host-side config / error logic mirrors the
reference (envkit.py:56-75, 461-481; dynamics.py:62-69)."""

import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "deskrl_b200.h")).read()
    return sorted(set(re.findall(r"\b(dk_[a-z0-9_]+)\s*\(", hdr)))


def test_header_symbols_exported_and_bound():
    from paper_2502_08844_b200 import _native

    lib = _native.lib()  # loads on a CPU-only host (static cudart)
    declared = _declared_symbols()
    assert len(declared) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (dk_[a-z0-9_]+)", out))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert sorted(_native.EXPORTED_SYMBOLS) == declared
    for s in declared:
        assert getattr(lib, s) is not None
    assert lib.dk_abi_version() == 7


def test_task_ids_and_dims():
    import ctypes

    from paper_2502_08844_b200 import _native

    lib = _native.lib()
    dims = {}
    for name in ("pendulum-swingup", "cartpole-balance", "acrobot-swingup", "reacher-easy"):
        t = lib.dk_task_id(name.encode())
        a, o, i = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        assert lib.dk_task_dims(t, ctypes.byref(a), ctypes.byref(o), ctypes.byref(i)) == 0
        dims[name] = (a.value, o.value, i.value)
    assert dims == {"pendulum-swingup": (1, 3, 1), "cartpole-balance": (1, 5, 3),
                    "acrobot-swingup": (1, 6, 1), "reacher-easy": (2, 10, 1)}
    assert lib.dk_task_id(b"go1-joystick") == -1


def test_create_without_gpu_reports_backend_error():
    import torch

    import paper_2502_08844_b200 as p

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(p.BackendError, match="CUDA"):
        p.BatchEnv(p.EnvConfig(), 4)


def test_config_validation_mirrors_reference(golden):
    import paper_2502_08844_b200 as p

    want = dict((k.split("/")[1], tuple(golden[k])) for k in golden.files if k.startswith("err/"))
    assert ",".join(p.registered_tasks()) == want["registered_tasks"][1]
    with pytest.raises(p.ConfigError) as e:
        p.resolve_task(p.EnvConfig(task="go1-joystick"))
    assert str(e.value) == want["unknown_task"][1]
    with pytest.raises(p.ConfigError, match="episode_length must be positive"):
        p.EnvConfig(episode_length=0)
    with pytest.raises(p.ConfigError, match="action_repeat must be >= 1"):
        p.EnvConfig(action_repeat=0)
    with pytest.raises(p.ConfigError, match="unknown obs_mode"):
        p.EnvConfig(obs_mode="rgb")
    with pytest.raises(p.InvalidInputError, match="dt must be positive"):
        p.DynamicsParams(dt=0)
    with pytest.raises(p.InvalidInputError, match="pole_mass must be positive"):
        p.DynamicsParams(pole_mass=-1)
    with pytest.raises(p.ConfigError, match="no pixel variant"):
        p.resolve_task(p.EnvConfig(task="reacher-easy-pixels"))
    spec = p.resolve_task(p.EnvConfig(task="reacher-easy"))
    assert spec.params.dt == 0.005 and spec.action_dim == 2 and spec.obs_dim == 10
    spec = p.resolve_task(p.EnvConfig(task="pendulum-swingup", dt=0.02),
                          p.DynamicsParams(pend_mass=2.0))
    assert spec.params.dt == 0.02 and spec.params.pend_mass == 2.0
    # error classes have the reference's bases
    assert issubclass(p.ConfigError, ValueError) and issubclass(p.InvalidInputError, ValueError)
    assert issubclass(p.UsageError, RuntimeError)


def test_reference_config_objects_are_accepted():
    """Duck-typed: anything with the EnvConfig / DynamicsParams attributes."""
    import paper_2502_08844_b200 as p

    class RefCfg:
        task, episode_length, action_repeat, dt, obs_mode = "acrobot-swingup", 5, 1, None, "state"
        seed, image_size, wide_init = 0, 64, False

    spec = p.resolve_task(RefCfg())
    assert spec.id == "acrobot-swingup" and spec.params.dt == 0.01


def test_infos_view():
    from paper_2502_08844_b200.envkit import _Infos

    info = np.arange(6, dtype=float).reshape(2, 3)
    mask = np.array([False, True])
    term = np.ones((2, 5))
    infos = _Infos(("upright", "centered", "still"), info, mask, term)
    assert len(infos) == 2
    assert infos[0] == {"upright": 0.0, "centered": 1.0, "still": 2.0}
    assert set(infos[1]) == {"upright", "centered", "still", "terminal_observation"}
    assert set(infos[-1]["terminal_observation"]) == {"state", "privileged_state"}
    assert [d.get("terminal_observation") is None for d in infos] == [True, False]


def test_ppo_struct_layouts_match_the_header():
    """ctypes mirrors of the PPO structs: sizes as the C compiler lays them out
    (capi_ppo.cu static_asserts sizeof(dk_ppo_post) == 192) and field offsets at
    natural alignment."""
    import ctypes

    from paper_2502_08844_b200 import _native as nat

    assert ctypes.sizeof(nat.PpoPostC) == 192
    assert nat.PpoPostC.reward_scaling.offset == 104
    assert nat.PpoPostC.next_val.offset == 184
    assert ctypes.sizeof(nat.PpoNormC) == 32
