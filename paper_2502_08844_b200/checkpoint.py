"""DSKRLCK1 checkpoints (ppo.py:592-684), interchangeable with the reference's
(SURVEY.md §8f rank 3): a checkpoint written by deskrl loads into the B200
rollout networks and DeviceRunningNormalizers, and one written here loads into
deskrl's TrainerState, byte for byte the same file for the same contents.

Layout: b"DSKRLCK1", u32 header length, JSON header {"format_version": 1,
"config_hash", "tensors": [{"name", "shape"}], "extra"}, the policy then value
state_dict tensors as little-endian float32 in header order, and -- when any
normaliser exists -- a JSON trailer {"policy"/"value": {"dim", "count", "mean",
"var"}} followed by its u32 length.
"""

from __future__ import annotations

import json
import struct

import numpy as np

from .envkit import ConfigError

MAGIC = b"DSKRLCK1"


def _norm_json(n):
    count, mean, var = (n.to_numpy() if hasattr(n, "to_numpy")
                        else (n.count, np.asarray(n.mean), np.asarray(n.var)))
    return {"dim": int(n.dim), "count": count, "mean": np.asarray(mean).tolist(),
            "var": np.asarray(var).tolist()}


def save_checkpoint(path, policy, value, config_hash: str, extra: dict | None = None,
                    policy_normalizer=None, value_normalizer=None):
    """Write ``policy`` / ``value`` (torch modules, any device) and the
    normalisers (DeviceRunningNormalizer or the reference's RunningNormalizer)."""
    tensors, blobs = [], []
    for prefix, module in (("policy", policy), ("value", value)):
        for name, param in module.state_dict().items():
            arr = param.detach().cpu().numpy().astype("<f4")
            tensors.append({"name": f"{prefix}.{name}", "shape": list(arr.shape)})
            blobs.append(arr.tobytes())
    header = json.dumps({"format_version": 1, "config_hash": config_hash, "tensors": tensors,
                         "extra": extra or {}}).encode()
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<I", len(header)))
        f.write(header)
        for blob in blobs:
            f.write(blob)
        if policy_normalizer is not None or value_normalizer is not None:
            norm = {}
            for key, n in (("policy", policy_normalizer), ("value", value_normalizer)):
                if n is not None:
                    norm[key] = _norm_json(n)
            trailer = json.dumps(norm).encode()
            f.write(trailer)
            f.write(struct.pack("<I", len(trailer)))


def read_checkpoint_header(path) -> dict:
    with open(path, "rb") as f:
        if f.read(8) != MAGIC:
            raise ConfigError("not a deskrl checkpoint")
        (hlen,) = struct.unpack("<I", f.read(4))
        return json.loads(f.read(hlen))


def load_checkpoint(path, policy, value, config_hash: str | None = None, device=None):
    """Load the tensors into ``policy`` / ``value``; returns (header,
    policy normaliser, value normaliser) -- DeviceRunningNormalizers (on
    ``device``) or None.  ``config_hash`` given: enforce it (strict_hash)."""
    import torch

    from .ppo import DeviceRunningNormalizer

    with open(path, "rb") as f:
        data = f.read()
    if data[:8] != MAGIC:
        raise ConfigError("not a deskrl checkpoint")
    (hlen,) = struct.unpack("<I", data[8:12])
    header = json.loads(data[12:12 + hlen])
    if header["format_version"] != 1:
        raise ConfigError(f"unsupported checkpoint version {header['format_version']}")
    if config_hash is not None and header["config_hash"] != config_hash:
        raise ConfigError("checkpoint config hash mismatch")
    offset = 12 + hlen
    loaded = {"policy": {}, "value": {}}
    for spec in header["tensors"]:
        count = int(np.prod(spec["shape"])) if spec["shape"] else 1
        arr = np.frombuffer(data, dtype="<f4", count=count, offset=offset).reshape(spec["shape"])
        offset += count * 4
        prefix, name = spec["name"].split(".", 1)
        loaded[prefix][name] = torch.as_tensor(arr.copy())
    policy.load_state_dict(loaded["policy"])
    value.load_state_dict(loaded["value"])
    norms = {"policy": None, "value": None}
    if offset < len(data):
        (tlen,) = struct.unpack("<I", data[-4:])
        norm = json.loads(data[len(data) - 4 - tlen:len(data) - 4])
        for key in norms:
            if key in norm:
                n = norm[key]
                norms[key] = DeviceRunningNormalizer(n["dim"], device=device, count=n["count"],
                                                     mean=np.array(n["mean"]),
                                                     var=np.array(n["var"]))
    return header, norms["policy"], norms["value"]


__all__ = ["MAGIC", "load_checkpoint", "read_checkpoint_header", "save_checkpoint"]
