"""ctypes binding of the C ABI in include/deskrl_b200.h (libdeskrl_b200.so).

There is no fallback: if the sm_100a library is missing this raises at import
of the env classes, so a GPU run can never silently fall back to CPU code.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DK_LIB_PATH: developer hook to load an experimental build (tools/exp_variants.sh);
# the default is the in-tree library.
LIB_PATH = os.environ.get("DK_LIB_PATH") or os.path.join(_HERE, "libdeskrl_b200.so")

DK_OK, DK_ERR_CONFIG, DK_ERR_INVALID_INPUT, DK_ERR_USAGE, DK_ERR_CUDA = range(5)
DK_F32, DK_F64 = 0, 1

# DynamicsParams field order (dynamics.py:40-60)
PARAM_FIELDS = (
    "dt", "gravity", "pend_mass", "pend_length", "pend_damping", "pend_torque_limit",
    "cart_mass", "pole_mass", "pole_length", "rail_limit", "cart_force_limit",
    "link1_mass", "link2_mass", "link1_length", "link2_length", "link_damping",
    "elbow_torque_limit", "reacher_torque_limit",
)


class DynamicsParamsC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in PARAM_FIELDS]


class EnvConfigC(ctypes.Structure):
    _fields_ = [
        ("task", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("episode_length", ctypes.c_int64),
        ("action_repeat", ctypes.c_int64),
        ("wide_init", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
    ]


REWARD_FIELDS = ("w_lin_vel", "sigma_lin_vel", "w_ang_vel", "sigma_ang_vel", "w_airtime",
                 "airtime_min", "airtime_max", "w_clearance", "w_phase", "sigma_phase",
                 "swing_height", "w_slip", "w_orientation", "w_torque", "w_joint_pos",
                 "w_action_rate", "w_energy", "w_pose", "w_termination", "w_standstill",
                 "w_lin_vel_z", "w_ang_vel_xy")
FRAME_FIELDS = ("base_orientation", "base_lin_vel", "base_ang_vel", "joint_pos", "joint_vel",
                "joint_torque", "foot_height", "foot_height_des", "foot_vel_xy", "foot_contact",
                "airtime", "touchdown", "phase", "command", "action", "prev_action",
                "joint_nominal", "joint_default", "done")


class PpoNormC(ctypes.Structure):
    """dk_ppo_norm (include/deskrl_b200.h)"""
    _fields_ = [("mean", ctypes.c_void_p), ("var", ctypes.c_void_p), ("epsilon", ctypes.c_double),
                ("copy", ctypes.c_int32), ("present", ctypes.c_int32)]


class PpoPostC(ctypes.Structure):
    """dk_ppo_post (include/deskrl_b200.h)"""
    _fields_ = [("n", ctypes.c_int64), ("dp", ctypes.c_int32), ("dv", ctypes.c_int32),
                ("action_dim", ctypes.c_int32), ("reserved", ctypes.c_int32)] + [
        (f, ctypes.c_void_p) for f in ("done", "trunc", "terminal_mask", "terminal_obs",
                                       "val_term", "count", "pos", "dones", "reward",
                                       "action")] + [
        ("reward_scaling", ctypes.c_double), ("discounting", ctypes.c_double)] + [
        (f, ctypes.c_void_p) for f in ("rewards_out", "actions_out", "reward_partial",
                                       "next_obs_p", "next_obs_v", "next_raw_p", "next_raw_v",
                                       "next_pol", "next_val")]


class RewardConfigC(ctypes.Structure):
    _fields_ = [(f, ctypes.c_double) for f in REWARD_FIELDS] + [
        ("standstill_gated", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class LocoFramesC(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in FRAME_FIELDS] + [
        ("nominal_stride", ctypes.c_int64), ("default_stride", ctypes.c_int64)]


class LocoOutputsC(ctypes.Structure):
    _fields_ = [(f, ctypes.c_void_p) for f in ("total", "unclipped", "terms", "state_obs",
                                              "privileged_obs")]


class NoiseKeyC(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("env_index_offset", ctypes.c_int64),
                ("episode", ctypes.c_void_p), ("step", ctypes.c_uint64)]


class VisualBoundsC(ctypes.Structure):
    _fields_ = [("nominal", ctypes.c_double * 13), ("color_jitter", ctypes.c_double),
                ("camera_offset_range", ctypes.c_double), ("zoom_range", ctypes.c_double * 2),
                ("brightness_range", ctypes.c_double * 2)]


_vp = ctypes.c_void_p
_u8p = ctypes.c_void_p
_i64 = ctypes.c_int64

_SIGS = {
    "dk_abi_version": (ctypes.c_int, []),
    "dk_stream_gate": (ctypes.c_int, [_vp, _i64, _vp]),
    "dk_phys_default_model": (ctypes.c_int, [_vp]),
    "dk_phys_create": (ctypes.c_int, [_vp, ctypes.c_int, _i64, ctypes.c_int, ctypes.POINTER(_vp)]),
    "dk_phys_destroy": (ctypes.c_int, [_vp]),
    "dk_phys_set_state": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "dk_phys_get_state": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "dk_phys_step": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp]),
    "dk_phys_inspect": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "dk_phys_check": (ctypes.c_int, [_vp]),
    "dk_phys_kernel_launches": (ctypes.c_int64, [_vp]),
    "dk_go1_default_config": (ctypes.c_int, [_vp]),
    "dk_go1_create": (ctypes.c_int, [_vp, _vp, ctypes.c_int, _i64, _i64, ctypes.c_int,
                                     ctypes.POINTER(_vp)]),
    "dk_go1_destroy": (ctypes.c_int, [_vp]),
    "dk_go1_reset": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_uint64, _vp, _vp, _vp]),
    "dk_go1_step": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _u8p, _u8p, _vp, _vp, _u8p,
                                   _vp]),
    "dk_go1_step_ex": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _u8p, _u8p, _vp, _vp, _vp,
                                      _u8p, _vp]),
    "dk_go1_get_state": (ctypes.c_int, [_vp] + [_vp] * 9 + [_vp]),
    "dk_go1_check": (ctypes.c_int, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "dk_go1_kernel_launches": (ctypes.c_int64, [_vp]),
    "dk_go1_get_params": (ctypes.c_int, [_vp, _vp, _vp]),
    "dk_mlp_pack": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]),
    "dk_mlp_forward": (ctypes.c_int, [_vp, _i64, _vp, _i64, _vp, _i64, _vp]),
    "dk_mlp_forward_dbg": (ctypes.c_int, [_vp, _i64, _vp, _i64, _vp, _i64, ctypes.c_int, _vp]),
    "dk_mlp_forward_count": (ctypes.c_int, [_vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp]),
    "dk_mlp_forward_pair": (ctypes.c_int, [_vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64,
                                           _vp, _i64, _vp]),
    "dk_last_error": (ctypes.c_char_p, []),
    "dk_task_id": (ctypes.c_int, [ctypes.c_char_p]),
    "dk_task_dims": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                    ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    "dk_env_create": (ctypes.c_int, [ctypes.POINTER(EnvConfigC), ctypes.POINTER(DynamicsParamsC),
                                     _i64, _i64, ctypes.c_int, ctypes.POINTER(_vp)]),
    "dk_env_destroy": (ctypes.c_int, [_vp]),
    "dk_env_reset": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_uint64, _vp, _vp]),
    "dk_env_step": (ctypes.c_int, [_vp, _vp, ctypes.c_int, _vp, _vp, _u8p, _u8p, _vp, _u8p, _vp,
                                   _vp]),
    "dk_env_rollout": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _u8p, _u8p, _vp, _u8p, _vp, _vp]),
    "dk_env_reset_host": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_uint64, _vp]),
    "dk_env_step_host": (ctypes.c_int, [_vp, _vp, ctypes.c_int, _vp, _vp, _u8p, _u8p, _vp, _u8p,
                                        _vp]),
    "dk_env_rollout_host": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, _vp, _u8p, _u8p, _vp, _u8p,
                                           _vp]),
    "dk_env_check_error": (ctypes.c_int, [_vp, _vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "dk_env_get_state": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _u8p]),
    "dk_env_set_state": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _u8p]),
    "dk_env_kernel_launches": (ctypes.c_int64, [_vp]),
    "dk_loco_tail": (ctypes.c_int, [ctypes.c_int, _i64, _i64, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(RewardConfigC), ctypes.POINTER(LocoFramesC),
                                    _vp, _vp, _vp, ctypes.POINTER(NoiseKeyC), _vp,
                                    ctypes.POINTER(LocoOutputsC), _vp, _vp]),
    "dk_loco_pd": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp,
                                  _vp, _vp, _vp]),
    "dk_loco_phase": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_int, _vp, _vp, _vp, _vp, _vp,
                                     _vp]),
    "dk_loco_progress_clip": (ctypes.c_int, [ctypes.c_int, _i64, _vp, _vp, _vp, _vp]),
    "dk_dr_sensor_noise": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_int, _vp, ctypes.c_int,
                                          _vp, _vp, _vp, _vp, ctypes.POINTER(NoiseKeyC), _vp]),
    "dk_dr_randomize_params": (ctypes.c_int, [_i64, ctypes.c_int, _vp, ctypes.c_int, _vp, _vp,
                                              _vp, _vp, ctypes.POINTER(NoiseKeyC), _vp, _vp,
                                              _vp]),
    "dk_dr_delay_reset": (ctypes.c_int, [_i64, ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(NoiseKeyC), _vp, _vp, _vp, _vp]),
    "dk_dr_delay_push_pop": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _vp,
                                            ctypes.POINTER(NoiseKeyC), _vp, _vp, _vp]),
    "dk_dr_pose_injection": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_int, _vp, _vp,
                                            ctypes.c_double, ctypes.POINTER(NoiseKeyC), _vp,
                                            _vp]),
    "dk_dr_curriculum": (ctypes.c_int, [_i64, _vp, _vp, _i64, _i64, _vp]),
    "dk_pixels_render_rgb": (ctypes.c_int, [_i64, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                            _vp, _vp, ctypes.c_int, _vp, _vp]),
    "dk_pixels_advance": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_int, _vp, _vp, ctypes.c_int,
                                         _vp, _vp, _vp, ctypes.c_int,
                                         ctypes.POINTER(VisualBoundsC), ctypes.c_uint64, _i64,
                                         ctypes.c_int, _vp]),
    "dk_pixels_stack": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_double, _vp, _vp, _vp, _vp]),
    "dk_pixels_terminal": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_int, _vp, _vp, _vp, _vp, _vp,
                                          _vp]),
    "dk_pixels_normalize": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _i64, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp,
                                           _vp, _vp]),
    "dk_ppo_sample": (ctypes.c_int, [_i64, ctypes.c_int, _vp, _vp, _i64, _vp, _vp, _vp, _vp,
                                     _vp, _vp]),
    "dk_ppo_gae": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _vp, _vp, _vp, _vp, ctypes.c_double,
                                  ctypes.c_double, _vp, _vp, _vp]),
    "dk_ppo_step_inputs": (ctypes.c_int, [_i64, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _vp,
                                          _vp, _vp, _vp, _vp, _vp, _vp]),
    "dk_ppo_step_bootstrap": (ctypes.c_int, [_i64, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp,
                                             _vp, _vp, _vp, _vp]),
    "dk_ppo_step_bootstrap_acc": (ctypes.c_int, [_i64, ctypes.c_int, _vp, _vp, _vp, _vp, _vp,
                                                 _vp, _vp, _vp, _vp, _vp]),
    "dk_ppo_boot_fixup": (ctypes.c_int, [_i64, _vp, _vp, ctypes.c_double, _vp, _vp]),
    "dk_ppo_step_post": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "dk_ppo_record_blocks": (_i64, [_i64]),
    "dk_ppo_step_record": (ctypes.c_int, [_i64, ctypes.c_int, _vp, _vp, _vp, _vp, _vp,
                                          ctypes.c_double, ctypes.c_double, _vp, _vp, _vp, _vp,
                                          _vp]),
    "dk_norm_update": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_int, _vp, ctypes.c_double,
                                      _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "dk_norm_workspace_bytes": (ctypes.c_size_t, [_i64, ctypes.c_int]),
    "dk_norm_colsum": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_int, _vp, _vp, _vp, _vp,
                                      ctypes.c_size_t, _vp]),
    "dk_norm_merge": (ctypes.c_int, [ctypes.c_int, ctypes.c_double, ctypes.c_double, _vp, _vp,
                                     _vp, _vp, _vp]),
    "dk_norm_apply": (ctypes.c_int, [ctypes.c_int, _i64, ctypes.c_int, _vp, ctypes.c_double,
                                     _vp, _vp, ctypes.c_double, ctypes.c_int, _vp, _vp]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def lib() -> ctypes.CDLL:
    """Load libdeskrl_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the sm_100a library first "
                "(python -m paper_2502_08844_b200.build or __graft_entry__.build())")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().dk_last_error()
    return msg.decode() if msg else ""
