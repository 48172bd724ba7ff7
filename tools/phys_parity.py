"""Parity report of the B200 articulated physics step (csrc/physics.cuh) against
the fp64 oracle (oracle/physics.c): inspection quantities, one step from
identical states, and a 100-step horizon, f64 and f32, feet-only and full
collision.  Writes gpurun_out/phys_parity.json.

    python tools/phys_parity.py [--n 8192]
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(a, b, floor):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float((np.abs(a - b) / np.maximum(np.abs(b), floor)).max()) if a.size else 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "phys_parity.json"))
    args = ap.parse_args()
    import torch

    from oracle import physics as op
    from paper_2502_08844_b200 import physics as P
    from paper_2502_08844_b200 import physmodel as pm

    n = args.n
    rep = {}
    for cfgname, kw in (("feet", {}), ("full", dict(collide_box=1, collide_thigh=1))):
        model = pm.go1_model(**kw)
        mc = model.to_c()
        qpos, qvel, ctrl = op.random_states(n, seed=7)
        if cfgname == "full":
            qpos[: n // 4, 2] = np.random.default_rng(9).uniform(0.02, 0.12, n // 4)
        ins_ref = op.inspect(mc, qpos, qvel)
        one = op.step(mc, qpos, qvel, ctrl, 1)
        for dtype in ("float64", "float32"):
            key = f"{cfgname}/{dtype}"
            r = {}
            sim = P.DevicePhysics(model, n, dtype=dtype)
            cast = lambda x: torch.as_tensor(x, device="cuda", dtype=sim.dtype)  # noqa: E731
            q32 = qpos.astype(np.float32).astype(np.float64) if dtype == "float32" else qpos
            v32 = qvel.astype(np.float32).astype(np.float64) if dtype == "float32" else qvel
            c32 = ctrl.astype(np.float32).astype(np.float64) if dtype == "float32" else ctrl
            ins_r = op.inspect(mc, q32, v32) if dtype == "float32" else ins_ref
            one_r = op.step(mc, q32, v32, c32, 1) if dtype == "float32" else one
            sim.set_state(cast(q32), cast(v32))
            ins = {k: v.double().cpu().numpy() for k, v in sim.inspect().items()}
            for k in ("M", "qfrc_bias", "xpos", "xipos"):
                d = np.abs(ins[k] - ins_r[k])
                r[f"inspect/{k}/abs"] = float(d.max())
                r[f"inspect/{k}/rel@1e-3"] = rel(ins[k], ins_r[k], 1e-3)
            out = sim.step(cast(c32), 1)
            sim.check()
            qp, qv = (x.double().cpu().numpy() for x in sim.state())
            o = {k: v.cpu().numpy() for k, v in out.items()}
            r["step1/ncon_equal_frac"] = float((o["ncon"] == one_r["ncon"]).mean())
            r["step1/geom_equal_frac"] = float(
                (o["contact_geom"] == one_r["contact_geom"]).all(axis=(1, 2)).mean())
            r["step1/ncon_mean"] = float(one_r["ncon"].mean())
            r["step1/solver_iter_mean"] = float(o["solver_iter"].mean())
            r["step1/solver_iter_ref_mean"] = float(one_r["solver_iter"].mean())
            r["step1/solver_iter_equal_frac"] = float((o["solver_iter"] == one_r["solver_iter"]).mean())
            same = (o["contact_geom"] == one_r["contact_geom"]).all(axis=(1, 2))
            for k, a, b in (("qpos", qp, one_r["qpos"]), ("qvel", qv, one_r["qvel"]),
                            ("qacc", o["qacc"], one_r["qacc"]),
                            ("qfrc_bias", o["qfrc_bias"], one_r["qfrc_bias"]),
                            ("qfrc_constraint", o["qfrc_constraint"], one_r["qfrc_constraint"]),
                            ("act_force", o["act_force"], one_r["act_force"]),
                            ("contact_dist", o["contact_dist"], one_r["contact_dist"]),
                            ("contact_force", o["contact_force"], one_r["contact_force"]),
                            ("sensordata", o["sensordata"], one_r["sensordata"])):
                a, b = np.asarray(a, np.float64)[same], np.asarray(b, np.float64)[same]
                r[f"step1/{k}/abs"] = float(np.abs(a - b).max()) if a.size else 0.0
                r[f"step1/{k}/rel@1e-3"] = rel(a, b, 1e-3)
            # normwise per world: ||d||_inf / max(||ref||_inf, 1)
            for k, a, b in (("qpos", qp, one_r["qpos"]), ("qvel", qv, one_r["qvel"]),
                            ("qacc", o["qacc"], one_r["qacc"])):
                nw = np.abs(a - b).max(1) / np.maximum(np.abs(b).max(1), 1.0)
                r[f"step1/{k}/normwise_max"] = float(nw.max())
                r[f"step1/{k}/normwise_p99"] = float(np.percentile(nw, 99))
            # 100 steps (ctrl held), from the same state
            sim.set_state(cast(q32), cast(v32))
            qp_r, qv_r = q32.copy(), v32.copy()
            ncon_eq, worst = [], {"qpos": [], "qvel": []}
            o100 = None
            for s in range(100):
                o100 = sim.step(cast(c32), 1)
                ref = op.step(mc, qp_r, qv_r, c32, 1)
                qp_r, qv_r = ref["qpos"], ref["qvel"]
                ncon_eq.append(float((o100["ncon"].cpu().numpy() == ref["ncon"]).mean()))
                if s in (0, 9, 99):
                    qp, qv = (x.double().cpu().numpy() for x in sim.state())
                    for k, a, b in (("qpos", qp, qp_r), ("qvel", qv, qv_r)):
                        nw = np.abs(a - b).max(1) / np.maximum(np.abs(b).max(1), 1.0)
                        r[f"h{s + 1}/{k}/normwise_p50"] = float(np.percentile(nw, 50))
                        r[f"h{s + 1}/{k}/normwise_p99"] = float(np.percentile(nw, 99))
                        r[f"h{s + 1}/{k}/normwise_max"] = float(nw.max())
                        r[f"h{s + 1}/{k}/frac_over_1e-3"] = float((nw > 1e-3).mean())
                    r[f"h{s + 1}/qpos/abs"] = float(np.abs(qp - qp_r).max())
                    r[f"h{s + 1}/qvel/abs"] = float(np.abs(qv - qv_r).max())
                    r[f"h{s + 1}/qpos/rel@1e-3"] = rel(qp, qp_r, 1e-3)
                    r[f"h{s + 1}/qvel/rel@1e-3"] = rel(qv, qv_r, 1e-3)
                    r[f"h{s + 1}/qvel/p99_abs"] = float(np.percentile(np.abs(qv - qv_r).max(1), 99))
            sim.check()
            if dtype == "float32":
                # the float64 oracle's own sensitivity: state rounded to float32
                # after every step (storage alone), against the exact oracle
                qe, ve, qx, vx = q32.copy(), v32.copy(), q32.copy(), v32.copy()
                for s in range(100):
                    e = op.step(mc, qe, ve, c32, 1)
                    qe = e["qpos"].astype(np.float32).astype(np.float64)
                    ve = e["qvel"].astype(np.float32).astype(np.float64)
                    x = op.step(mc, qx, vx, c32, 1)
                    qx, vx = x["qpos"], x["qvel"]
                    if s in (0, 9, 99):
                        for k, a, b in (("qpos", qe, qx), ("qvel", ve, vx)):
                            nw = np.abs(a - b).max(1) / np.maximum(np.abs(b).max(1), 1.0)
                            r[f"envelope_h{s + 1}/{k}/normwise_p99"] = float(np.percentile(nw, 99))
                            r[f"envelope_h{s + 1}/{k}/normwise_max"] = float(nw.max())
                            r[f"envelope_h{s + 1}/{k}/frac_over_1e-3"] = float((nw > 1e-3).mean())
            r["h100/ncon_equal_frac_min"] = float(min(ncon_eq))
            r["h100/ncon_equal_frac_mean"] = float(np.mean(ncon_eq))
            rep[key] = r
            print(key, json.dumps({k: (f"{v:.3g}" if isinstance(v, float) else v)
                                   for k, v in r.items()}), flush=True)
            sim.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(rep, f, indent=1)


if __name__ == "__main__":
    main()
