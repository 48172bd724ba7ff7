"""Benchmark of the batched env step (the reference's hot path) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU)

Headline (BASELINE.json's metric): physics steps/s of the Go1 joystick env at
8192 worlds per GPU.  A "step" is one control step of every world through the
fused kernel (csrc/go1env.cuh): action -> PD targets, 5 physics steps (FK, CRB
mass matrix, contacts, Newton solver, Euler), reward, noisy observation,
termination and Philox auto-reset; physics steps = control steps x 5 (the
metric's physics steps, as the reference counts env-steps x action_repeat,
SURVEY.md §8d).  K steps run as ceil(K / --unroll) fused launches over a ring
of action / output chunks, behind a device gate (dk_stream_gate) so the CUDA
events time the device, not host submission.  Rank r owns global worlds
[r*N, (r+1)*N) -- no collective on the data path ("weak" scaling).

The reference has no Go1 physics: parity is against the repo's
independent oracle (UNPINNED), and the CPU baseline / --impl reference arm is
that oracle's C physics step on all host cores (kind "port").  The analytic
tasks the reference does implement (cartpole etc., pinned bit-exact in f64)
are timed on their own lines before the headline (extra "cartpole", "sweep",
"all_tasks", ...), each a JSON line without a top-level "metric" key.

Prints the headline JSON line (rank 0) LAST, with roofline, cpu_baseline,
an end-to-end number through the public API with host buffers, the float64
leg and the clocks seen around the timed region.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import platform
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "physics steps/sec (Go1 joystick, 8192 worlds/GPU) at 1/2/4/8 B200 vs CPU host"
ANALYTIC_METRIC = "physics steps/sec (8192 worlds/GPU) at 1/2/4/8 B200 vs CPU host"
GO1 = "go1-joystick"
GO1_SUBSTEPS = 5
UNIT = "physics_steps/s"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--task", default=GO1, help="go1-joystick (headline) or an analytic task")
    ap.add_argument("--analytic-task", default="cartpole-balance",
                    help="analytic task of the secondary 'cartpole' line")
    ap.add_argument("--analytic-steps", type=int, default=20_000,
                    help="steps of the secondary analytic line")
    ap.add_argument("--num-envs", type=int, default=8192, help="worlds per GPU")
    ap.add_argument("--dtype", default="float32", choices=["float32", "float64"])
    ap.add_argument("--unroll", type=int, default=0,
                    help="env steps fused per launch (0: 50 for go1, 1000 for analytic tasks)")
    ap.add_argument("--ring", type=int, default=6, help="action/output chunks in the ring")
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="steps of the e2e leg (0: 200 for go1, 20000 for analytic tasks)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tail", action="store_true", help="skip the Go1-shape step-tail line")
    ap.add_argument("--no-f64", action="store_true", help="skip the precision-matched f64 leg")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the drop-in BatchEnv.step and world-count sweep lines")
    a = ap.parse_args()
    if a.unroll <= 0:
        a.unroll = 50 if a.task == GO1 else 1000
    if a.e2e_steps <= 0:
        a.e2e_steps = 200 if a.task == GO1 else 20_000
    return a


# ---------------------------------------------------------------------------
# algorithmic bytes: per world-step and per launch


def bytes_per_world_step(A, O, I, esz):
    # action in; obs, reward, info out; done, trunc, terminal_mask flags out
    return esz * (A + O + 1 + I) + 3


def state_io_bytes(NS, esz):
    # per world per launch: state read + write, steps/episode/needs_reset read + write
    return 2 * (NS * esz + 4 + 4 + 1)


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML, the library nvidia-smi reads)


class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, device_index: int, period_s: float = 0.002):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._period = period_s
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = self._handle(pynvml, device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - no NVML
            self._nv = None
            self.error = str(e)

    @staticmethod
    def _handle(nv, device_index):
        """NVML handle of the CUDA device by PCI bus id (NVML's enumeration
        ignores CUDA_VISIBLE_DEVICES, so an index could name another GPU)."""
        try:
            import torch

            p = torch.cuda.get_device_properties(device_index)
            bus = f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(device_index)

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self._period)

    def start(self):
        return self.__enter__()

    def stop(self):
        self.__exit__(None, None, None)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        if self._nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.error}
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons - {"gpu_idle"}),
                "samples": len(self.samples)}


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(task, dtype, num_envs, unroll):
    """dram bytes per launch of the rollout kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            tab = json.load(f)
        return tab.get(f"{task}/{dtype}/{num_envs}/{unroll}")
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port of the reference algorithm on the host cores


def cpu_rate(task, num_envs, seconds, nthreads=0, steps=None):
    from oracle.oracle import ACTION_DIM, TASK_IDS, OracleBatchEnv, max_threads, use_all_host_threads

    use_all_host_threads()
    A = ACTION_DIM[TASK_IDS[task]]
    env = OracleBatchEnv(task, num_envs)
    env.reset(seed=0)
    rng = np.random.default_rng(0)
    threads = nthreads or max_threads()
    probe = 20
    acts = rng.uniform(-1, 1, (probe, num_envs, A))
    t0 = time.perf_counter()
    env.rollout(acts, nthreads=threads)
    dt = time.perf_counter() - t0
    if steps is None:
        steps = max(probe, int(seconds / max(dt / probe, 1e-9)))
    acts = rng.uniform(-1, 1, (min(steps, 2000), num_envs, A))
    done = 0
    t0 = time.perf_counter()
    while done < steps:
        k = min(steps - done, acts.shape[0])
        env.rollout(acts[:k], nthreads=threads)
        done += k
    dt = time.perf_counter() - t0
    return steps * num_envs / dt, threads, steps, dt


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor()


# ---------------------------------------------------------------------------


TASK_DIMS = {"cartpole-balance": (1, 5, 3), "pendulum-swingup": (1, 3, 1),
             "acrobot-swingup": (1, 6, 1), "reacher-easy": (2, 10, 1)}  # (A, O, info terms)


def headline_config(args, world, task=None, steps=None, unroll=None):
    """The `config` object of an analytic-task line."""
    task = task or args.task
    steps = args.steps if steps is None else steps
    A, O, I = TASK_DIMS[task]
    esz = 8 if args.dtype == "float64" else 4
    U = min(unroll or args.unroll, steps)
    R = max(2, args.ring)
    bpw = bytes_per_world_step(A, O, I, esz)
    chunk_mb = U * args.num_envs * (bpw + A * esz) / 1e6
    nlaunch = -(-steps // U)
    if nlaunch == 1:
        l2_note = "flushed before the timed region (a single launch)"
    else:
        l2_note = (f"flushed before the timed region; {R}-chunk ring of {chunk_mb:.0f} MB "
                   f"chunks ({'>' if chunk_mb * min(R, nlaunch) > 126 else '<'} 126 MB L2)")
    return {
        "workload": f"{task} BatchEnv.step (dynamics, reward + info terms, obs, "
                    "truncation, Philox autoreset), episode_length 1000",
        "task": task, "worlds_per_gpu": args.num_envs,
        "global_worlds": args.num_envs * world, "steps_per_launch": U,
        "parallelism": f"worlds sharded dp{world}",
        "l2": l2_note,
    }


def run_reference(args, rank, world):
    """The CPU arm: rank 0 alone times the oracle on all host cores (the
    reference itself has no Go1 physics and is single-threaded Python for the
    analytic tasks); other ranks exit without work."""
    if rank != 0:
        return
    from oracle.oracle import build as build_oracle

    build_oracle()
    if args.task == GO1:
        # warm-up, then exactly K control steps (x 5 physics steps) of every
        # world, bounded to ~30 s of CPU work
        cpu_go1_rate(args.num_envs, max(1, min(args.warmup, 2)), seconds=2.0)
        rate, threads, n_phys, dt = cpu_go1_rate(args.num_envs, args.steps, seconds=30.0)
        steps = n_phys / GO1_SUBSTEPS
        kind_note = ("oracle/physics.c, the independent fp64 restatement of the Go1 physics "
                     "step (the reference has no Go1 physics, SPEC.md:8); physics only, the "
                     "env tail excluded")
        cfg = go1_config_obj(args, world, min(args.unroll, args.steps))
        metric, dtype = METRIC, "f64"
    else:
        cpu_rate(args.task, args.num_envs, 0.5, steps=max(3, min(args.warmup, 200)))
        rate, threads, steps, dt = cpu_rate(args.task, args.num_envs, 0, steps=args.steps)
        kind_note = "oracle/oracle.c, the bit-exact C restatement of deskrl BatchEnv.step"
        cfg = headline_config(args, world)
        metric, dtype = ANALYTIC_METRIC, "f64"
    line = {
        "impl": "reference", "metric": metric, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / max(steps, 1e-9) * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{steps:g} env steps x {args.num_envs} worlds on {threads} "
                                   f"threads ({cpu_model()}) in {dt:.1f} s; {kind_note}"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        # what was actually timed: rank 0 alone, num_envs worlds on the host
        # cores, whatever N the job was launched with
        "timed_worlds": args.num_envs, "timed_ranks": 1,
    }
    print(json.dumps(line), flush=True)


class DeviceGate:
    """dk_stream_gate: the stream waits on a pinned host flag, so the timed
    region (events + launches) is fully enqueued before the device starts it
    and host submission latency stays outside the events."""

    def __init__(self):
        import torch

        from paper_2502_08844_b200 import _native

        self._lib = _native.lib()
        self.flag = torch.zeros(1, dtype=torch.int32, pin_memory=True)

    def close(self, stream):
        self.flag[0] = 0
        # ~5e6 polls (seconds) as a safety valve: the device never hangs on it
        rc = self._lib.dk_stream_gate(self.flag.data_ptr(), 5_000_000, stream.cuda_stream)
        if rc != 0:
            raise RuntimeError("dk_stream_gate failed")

    def open(self):
        self.flag[0] = 1


_GATE = None


def gated_region(fn, stream, dev):
    """Enqueue gate, start event, fn()'s launches, end event; release; return ms."""
    import torch

    global _GATE
    if _GATE is None:
        _GATE = DeviceGate()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _GATE.close(stream)
    t0.record(stream)
    fn()
    t1.record(stream)
    _GATE.open()
    torch.cuda.synchronize(dev)
    return t0.elapsed_time(t1)


def measure_rollout(args, dtype, dev, rank, world, dist, local_rank, task=None, steps=None,
                    unroll=None):
    """The headline measurement for one real type: W warm-up steps, L2 flush,
    then exactly K steps of every world as fused rollout launches, behind a
    device gate, timed with CUDA events on the launching stream, max over ranks."""
    import torch

    import paper_2502_08844_b200 as dk

    n = args.num_envs
    task = task or args.task
    steps = args.steps if steps is None else steps
    cfg = dk.EnvConfig(task=task)
    env = dk.DeviceBatchEnv(cfg, n, dtype=dtype, device=local_rank, env_index_offset=rank * n)
    A, O, I, NS = env.action_dim, env.obs_dim, len(env.info_keys), env.spec.state_dim
    tdt = env.dtype
    esz = 8 if tdt == torch.float64 else 4
    U = min(unroll or args.unroll, steps)
    R = max(2, args.ring)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    acts = [torch.rand((U, n, A), generator=gen, device=dev, dtype=tdt) * 2 - 1 for _ in range(R)]
    outs = [env._outputs((U,), True) for _ in range(R)]
    env.reset(seed=0)
    stream = torch.cuda.current_stream(dev)

    def launch(j, k):
        a = acts[j % R] if k == U else acts[j % R][:k]
        o = outs[j % R] if k == U else {kk: (v[:k] if v is not None else None)
                                         for kk, v in outs[j % R].items()}
        env.rollout(a, with_info=True, out=o)

    # warm-up
    w_left, j = args.warmup, 0
    while w_left > 0:
        k = min(U, w_left)
        launch(j, k)
        w_left -= k
        j += 1
    env.check()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush.zero_()  # evict L2 before the timed region
    torch.cuda.synchronize(dev)
    del flush

    nlaunch = (steps + U - 1) // U
    launches0 = env.kernel_launches
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)

    def region():
        left = steps
        for L in range(nlaunch):
            k = min(U, left)
            launch(j + L, k)  # back to back: events between launches cost 8% (measured)
            left -= k

    elapsed_ms = gated_region(region, stream, dev)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    env.check()
    gpu_launches = env.kernel_launches - launches0
    if dist is not None:
        t = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    total_steps = steps * n * world * cfg.action_repeat
    value = total_steps / (elapsed_ms / 1e3)

    # roofline of the rollout kernel (the only kernel of a launch)
    peak, peak_src = hbm_peak()
    bpw = bytes_per_world_step(A, O, I, esz)
    alg_bytes_launch = n * U * bpw + n * state_io_bytes(NS, esz) + n * (U // 1000) * O * esz
    # average launch duration over the timed region (device events around the
    # whole gated region / launches: includes any inter-launch gaps, so the
    # achieved bandwidth is a lower bound for the kernel itself)
    avg_launch_s = elapsed_ms / 1e3 * U / steps
    achieved = alg_bytes_launch / avg_launch_s / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_source": peak_src,
            "traffic": ncu_traffic(task, dtype, n, U),
            "kernel": "rollout_kernel", "alg_bytes_per_launch": alg_bytes_launch,
            "bytes_per_world_step": bpw, "avg_launch_ms": avg_launch_s * 1e3}
    return {"env": env, "value": value, "elapsed_ms": elapsed_ms, "gpu_launches": gpu_launches,
            "roofline": roof, "dims": (A, O, I, esz), "ms_per_step": elapsed_ms / steps}


# ---------------------------------------------------------------------------
# Go1 joystick (headline)

# algorithmic bytes per control step and world (float32): actions in; state
# obs, privileged obs, reward out; done / trunc / terminal-mask bytes out
GO1_BYTES_STEP = 4 * (12 + 56 + 75 + 1) + 3
# per launch and world: the env state read + written once (qpos 19, qvel 18,
# command 3, phase 4, airtime 4, prev_action 12 reals; last_contact 4 B,
# steps and episode 4 B each)
GO1_STATE_BYTES = 2 * (4 * (19 + 18 + 3 + 4 + 4 + 12) + 4 + 8)


def go1_config_obj(args, world, U):
    return {
        "workload": "Go1 joystick env step, one fused kernel (go1env.cuh): 5 physics steps "
                    "(CRB, contacts, Newton) + reward + obs + autoreset with per-world DR; "
                    "Go1-shaped model, 18 DoF, h=4ms; no reference impl (SPEC.md:8)",
        "task": GO1, "worlds_per_gpu": args.num_envs, "global_worlds": args.num_envs * world,
        "physics_steps_per_env_step": GO1_SUBSTEPS, "env_steps_per_launch": U,
        "parallelism": f"worlds sharded dp{world}",
        "l2": "flushed before the timed region; state on chip within a launch",
    }


def measure_go1(args, dtype, dev, rank, world, dist, local_rank, steps=None):
    import torch

    from paper_2502_08844_b200 import go1env as G

    n = args.num_envs
    steps = args.steps if steps is None else steps
    env = G.DeviceGo1Env(n, G.Go1Config(), dtype=dtype, device=local_rank,
                         env_index_offset=rank * n)
    U = min(args.unroll, steps)
    R = max(2, args.ring)
    gen = torch.Generator(device=dev)
    gen.manual_seed(4321 + rank)
    acts = [torch.rand((U, n, 12), generator=gen, device=dev, dtype=env.dtype) * 2 - 1
            for _ in range(R)]
    outs = [env.outputs(U) for _ in range(R)]
    env.reset(seed=0)
    stream = torch.cuda.current_stream(dev)

    def launch(j, k):
        o = outs[j % R] if k == U else {kk: (v[:k] if v is not None else None)
                                         for kk, v in outs[j % R].items()}
        env.rollout(acts[j % R][:k], out=o)

    w_left, j = args.warmup, 0
    while w_left > 0:
        k = min(U, w_left)
        launch(j, k)
        w_left -= k
        j += 1
    env.check()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush.zero_()
    torch.cuda.synchronize(dev)
    del flush
    nlaunch = (steps + U - 1) // U
    launches0 = env.kernel_launches
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)

    def region():
        left = steps
        for L in range(nlaunch):
            k = min(U, left)
            launch(j + L, k)
            left -= k

    elapsed_ms = gated_region(region, stream, dev)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    env.check()
    gpu_launches = env.kernel_launches - launches0
    if dist is not None:
        t = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    total = steps * n * world * GO1_SUBSTEPS
    value = total / (elapsed_ms / 1e3)
    esz = 8 if env.dtype == torch.float64 else 4
    bstep = GO1_BYTES_STEP if esz == 4 else 8 * (12 + 56 + 75 + 1) + 3
    bstate = GO1_STATE_BYTES if esz == 4 else 2 * (8 * (19 + 18 + 3 + 4 + 4 + 12) + 4 + 8)
    alg = n * U * bstep + n * bstate
    avg_launch_s = elapsed_ms / 1e3 * U / steps
    peak, src = hbm_peak()
    roof = {"bound": "hbm", "achieved": alg / avg_launch_s / 1e9, "peak": peak, "unit": "GB/s",
            "frac": alg / avg_launch_s / 1e9 / peak, "peak_source": src,
            "traffic": ncu_traffic(GO1, dtype, n, U), "kernel": "go1_env_kernel",
            "alg_bytes_per_launch": alg, "bytes_per_env_step": bstep,
            "avg_launch_ms": avg_launch_s * 1e3,
            "note": "compute/latency bound; see profiles/r02_ncu_go1.md",
            "compute": ncu_compute(GO1, dtype)}
    return {"env": env, "value": value, "elapsed_ms": elapsed_ms, "gpu_launches": gpu_launches,
            "roofline": roof, "ms_per_step": elapsed_ms / steps, "U": U,
            "env_steps_per_s": value / GO1_SUBSTEPS}


def ncu_compute(kernel_key, dtype):
    """issue / pipe utilisation of the kernel from the committed ncu capture"""
    path = os.path.join(ROOT, "profiles", "compute.json")
    try:
        with open(path) as f:
            return json.load(f).get(f"{kernel_key}/{dtype}")
    except Exception:
        return None


def measure_go1_e2e(env, args, dev, dist, world):
    """The same steps through the public API with HOST buffers: per chunk, the
    actions copied from pinned host memory, DeviceGo1Env.rollout, and the
    observations / rewards / flags copied back, all inside the timed region."""
    import torch

    n, K = env.num_envs, args.e2e_steps
    U = min(args.unroll, K, 10)  # short chunks: the pipeline fills / drains faster
    pin = lambda *s, d=env.dtype: torch.empty(s, dtype=d, pin_memory=True)  # noqa: E731
    acts_h = pin(K, n, 12)
    acts_h.copy_(torch.rand((K, n, 12), dtype=env.dtype) * 2 - 1)
    obs_h, priv_h, rew_h = pin(K, n, 56), pin(K, n, 75), pin(K, n)
    done_h, trunc_h = pin(K, n, d=torch.uint8), pin(K, n, d=torch.uint8)
    dev_out = [env.outputs(U, with_terminal=False) for _ in range(2)]
    dev_act = [torch.empty((U, n, 12), dtype=env.dtype, device=dev) for _ in range(2)]

    # Pipelined like a serving loop: chunk c+1's actions go up on one copy stream
    # and chunk c's outputs come down on another while chunk c+1 computes (two
    # device buffer sets; events guard their reuse).
    main = torch.cuda.current_stream(dev)
    up, down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_done, ev_copied = [None, None], [None, None]

    def run(k0, k1, slot):
        k = k1 - k0
        a = dev_act[slot][:k]
        with torch.cuda.stream(up):
            if ev_done[slot] is not None:
                up.wait_event(ev_done[slot])  # the slot's previous rollout has read its actions
            a.copy_(acts_h[k0:k1], non_blocking=True)
            ev_up = torch.cuda.Event()
            ev_up.record(up)
        main.wait_event(ev_up)
        if ev_copied[slot] is not None:
            main.wait_event(ev_copied[slot])  # the slot's previous outputs are on the host
        o = {kk: (v[:k] if v is not None else None) for kk, v in dev_out[slot].items()}
        env.rollout(a, out=o)
        ev_done[slot] = torch.cuda.Event()
        ev_done[slot].record(main)
        with torch.cuda.stream(down):
            down.wait_event(ev_done[slot])
            obs_h[k0:k1].copy_(o["obs"], non_blocking=True)
            priv_h[k0:k1].copy_(o["privileged_state"], non_blocking=True)
            rew_h[k0:k1].copy_(o["reward"], non_blocking=True)
            done_h[k0:k1].copy_(o["done"], non_blocking=True)
            trunc_h[k0:k1].copy_(o["trunc"], non_blocking=True)
            ev_copied[slot] = torch.cuda.Event()
            ev_copied[slot].record(down)

    run(0, min(U, K), 0)
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for c, k0 in enumerate(range(0, K, U)):
        run(k0, min(K, k0 + U), c % 2)
    torch.cuda.synchronize(dev)
    dt = time.perf_counter() - t0
    env.check()
    if dist is not None:
        t = torch.tensor([dt], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    esz = 8 if env.dtype == torch.float64 else 4
    return {"value": K * n * world * GO1_SUBSTEPS / dt, "unit": UNIT,
            "h2d_bytes_per_step": n * 12 * esz,
            "d2h_bytes_per_step": n * ((56 + 75 + 1) * esz + 2),
            "api": "paper_2502_08844_b200.go1env.DeviceGo1Env.rollout with pinned host "
                   "actions in and obs / privileged obs / reward / done / trunc out; "
                   "copies on two copy streams overlapping the next chunk's rollout",
            "steps": K, "chunk_steps": U}


def cpu_go1_rate(num_envs, steps, seconds=None):
    """The physics oracle (oracle/physics.c, fp64, OpenMP over worlds) on the
    host cores: physics steps/s of the Go1 model from the home pose with
    random PD targets.  Bounded: at most `seconds` of CPU work when given."""
    from oracle import physics as op
    from oracle.oracle import max_threads, use_all_host_threads
    from paper_2502_08844_b200 import physmodel as pm

    use_all_host_threads()
    m = pm.go1_model()
    mc = m.to_c()
    q, v = pm.home_qpos(num_envs), np.zeros((num_envs, 18))
    ctrl = q[:, 7:] + np.random.default_rng(0).uniform(-0.5, 0.5, (num_envs, 12))
    t0 = time.perf_counter()
    o = op.step(mc, q, v, ctrl, 2)
    probe = (time.perf_counter() - t0) / 2
    n_phys = steps * GO1_SUBSTEPS
    if seconds is not None:
        n_phys = max(2, min(n_phys, int(seconds / max(probe, 1e-9))))
    t0 = time.perf_counter()
    op.step(mc, o["qpos"], o["qvel"], ctrl, n_phys)
    dt = time.perf_counter() - t0
    return num_envs * n_phys / dt, max_threads(), n_phys, dt


def bench_go1_sweep(args, dev, sizes=(1024, 8192, 65536), K=50, reps=3):
    """Go1 joystick env (fused kernel) at several world counts, f32."""
    import torch

    from paper_2502_08844_b200 import go1env as G

    out = []
    for n in sizes:
        env = G.DeviceGo1Env(n, G.Go1Config(), dtype="float32", device=dev.index)
        env.reset(seed=0)
        acts = torch.rand((K, n, 12), device=dev) * 2 - 1
        o = env.outputs(K)
        env.rollout(acts, out=o)
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            env.rollout(acts, out=o)
        b.record()
        torch.cuda.synchronize(dev)
        env.check()
        s = a.elapsed_time(b) / 1e3 / reps
        out.append({"worlds": n, "physics_steps_per_s": n * K * GO1_SUBSTEPS / s,
                    "env_steps_per_s": n * K / s})
        env.close()
        del acts, o
    return out


def bench_phys_only(args, dev, K=100, reps=3):
    """The physics kernel alone (dk_phys_step, ctrl held, no tail), 8192 worlds,
    feet-only and full (trunk box + thigh capsules) collision, f32 and f64."""
    import torch

    from oracle import physics as op
    from paper_2502_08844_b200 import physics as P
    from paper_2502_08844_b200 import physmodel as pm

    res = {}
    n = args.num_envs
    for cfg, kw in (("feet", {}), ("full", dict(collide_box=1, collide_thigh=1))):
        for dt in ("float32", "float64"):
            sim = P.DevicePhysics(pm.go1_model(**kw), n, dtype=dt, device=dev.index)
            q, v, c = op.random_states(n, seed=1)
            tt = lambda x: torch.as_tensor(x, device=dev, dtype=sim.dtype)  # noqa: E731
            sim.set_state(tt(q), tt(v))
            ct = tt(c)
            sim.step(ct, K, diag=False)
            torch.cuda.synchronize(dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                sim.step(ct, K, diag=False)
            b.record()
            torch.cuda.synchronize(dev)
            sim.check()
            res[f"{cfg}/{dt}"] = n * K * reps / (a.elapsed_time(b) / 1e3)
            sim.close()
    return {"unit": UNIT, "worlds": n, "physics_steps_per_s": res,
            "note": "dk_phys_step: FK, CRB mass matrix, RNE, collision, Newton solver, Euler; "
                    "random states around the home pose"}


def emit_extra(name, obj):
    """Secondary results go on their own short lines BEFORE the headline line
    (no top-level "metric" key), so the headline stays the last line."""
    print(json.dumps({"extra": name, "result": obj}), flush=True)


def run_b200(args, rank, world, local_rank, dist):
    import torch

    from paper_2502_08844_b200 import _native

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if args.task != GO1:
        return run_b200_analytic(args, rank, world, local_rank, dist)
    n = args.num_envs
    # NVML clocks: sampled from before the warm-up until after the f64 leg
    clocks = ClockSampler(local_rank).start()
    head = measure_go1(args, args.dtype, dev, rank, world, dist, local_rank)
    other = "float64" if args.dtype == "float32" else "float32"
    f_other = None
    if not args.no_f64:
        r = measure_go1(args, other, dev, rank, world, dist, local_rank)
        r["env"].close()
        f_other = {"dtype": "f64" if other == "float64" else "f32", "value": r["value"],
                   "ms_per_step": r["ms_per_step"], "gpu_launches": r["gpu_launches"],
                   "roofline": {k: r["roofline"][k] for k in ("achieved", "frac", "avg_launch_ms")}}
    clocks.stop()
    env = head["env"]
    e2e = measure_go1_e2e(env, args, dev, dist, world) if args.e2e_steps > 0 else None

    extras = {}
    if rank == 0 and not args.no_extra:
        # the pinned analytic task (the reference's own physics) at the same world count
        # rank-0-only lines: no collective inside (the other ranks are not there)
        extras["cartpole"] = analytic_line(args, dev, 0, 1, None, local_rank)
        extras["go1_sweep"] = bench_go1_sweep(args, dev)
        extras["physics_only"] = bench_phys_only(args, dev)
        extras["loco_small"] = bench_loco_small(args, dev)
        extras["e2e_dropin_step"] = bench_dropin_step(args, dev)
        extras["sweep"] = bench_sweep(args, dev)
        extras["all_tasks"] = bench_tasks(args, dev)
        extras["ppo_rollout"] = bench_ppo_rollout(args, dev)
        extras["go1_ppo_rollout"] = bench_go1_ppo_rollout(args, dev)
        extras["pixels"] = bench_pixels(args, dev)
    if not args.no_tail:
        extras["go1_tail"] = bench_go1_tail(args, dev, rank)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            rate, threads, n_phys, dt = cpu_go1_rate(n, args.steps, seconds=args.cpu_seconds)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                   "sample": f"{n_phys} physics steps x {n} worlds in {dt:.1f}s on {threads} "
                             f"threads ({cpu_model()}); oracle/physics.c, the independent fp64 "
                             "restatement of the Go1 physics step (no reference "
                             "implementation exists); physics only, env tail excluded"}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "error": str(e)}

    if rank == 0:
        for k, v in extras.items():
            emit_extra(k, v)
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.dtype == "float32" else "f64",
            "data": "synthetic U(-1,1) actions in HBM; Go1-shaped model (no assets)",
            "config": go1_config_obj(args, world, head["U"]),
            "env_steps_per_s": head["env_steps_per_s"],
            "roofline": head["roofline"],
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": head["gpu_launches"],
            "f64" if other == "float64" else "f32": f_other,
            "cartpole": None if "cartpole" not in extras else {
                k: extras["cartpole"].get(k) for k in ("value", "frac", "f64_value", "e2e")},
            "clocks": clocks.summary(),
            "library": os.path.relpath(_native.LIB_PATH, ROOT),
            "extra_lines": sorted(extras),
        }
        print(json.dumps(line), flush=True)
    env.close()


REF_DIR = os.path.join(ROOT, "baseline", "_ref")
_REF_SNIPPET = (
    "import json, sys\n"
    "from deskrl import bench\n"
    "from deskrl.envkit import EnvConfig\n"
    "r = bench.measure_stage(bench.Stage.ENV_STEP, EnvConfig(task=sys.argv[1]), num_envs=1024,"
    " repetitions=int(sys.argv[2]), steps_per_batch=16)\n"
    "print(json.dumps({'sps': r.median_sps, 'lo': r.ci_low, 'hi': r.ci_high}))\n")


def reference_python_rate(task, procs=1, reps=10, timeout=120):
    """The UNMODIFIED reference (deskrl from baseline/_ref, installed with pip
    from /root/reference) timed by its own bench.measure_stage(ENV_STEP) on
    1024 worlds: one process, or `procs` independent
    processes whose rates are summed (its BatchEnv threads are GIL-bound)."""
    import subprocess

    if not os.path.isdir(os.path.join(REF_DIR, "deskrl")):
        return {"unavailable": "baseline/_ref not installed"}
    env = dict(os.environ, PYTHONPATH=REF_DIR, OMP_NUM_THREADS="1", CUDA_VISIBLE_DEVICES="")
    ps = [subprocess.Popen([sys.executable, "-c", _REF_SNIPPET, task, str(reps)], env=env,
                           stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
          for _ in range(procs)]
    rates = []
    for p in ps:
        try:
            out, _ = p.communicate(timeout=timeout)
            rates.append(json.loads(out.strip().splitlines()[-1])["sps"])
        except Exception as e:  # pragma: no cover
            p.kill()
            return {"error": str(e)}
    return {"value": float(sum(rates)), "unit": "env_steps/s", "processes": procs,
            "per_process": rates, "kind": "reference",
            "sample": f"deskrl.bench.measure_stage(ENV_STEP, {task}, 1024 worlds, {reps} "
                      "reps x 16 steps) per process, baseline/_ref (pip-installed reference)"}


def analytic_line(args, dev, rank, world, dist, local_rank):
    """The previous round's headline: the analytic task (cartpole, pinned
    bit-exact in f64 against the reference) at the bench's world count, gated,
    f32 + f64 legs and the host-buffer C-ABI e2e."""
    task, steps = args.analytic_task, args.analytic_steps
    r = measure_rollout(args, "float32", dev, rank, world, dist, local_rank, task=task,
                        steps=steps, unroll=1000)
    A, O, I, esz = r["dims"]
    e2e = measure_e2e(r["env"], args, dev, dist, A, O, I, esz, world, K=20_000, chunk=1000)
    r["env"].close()
    r64 = measure_rollout(args, "float64", dev, rank, world, dist, local_rank, task=task,
                          steps=steps, unroll=1000)
    r64["env"].close()
    ref1 = reference_python_rate(task, 1) if not args.no_cpu else None
    nproc = min(len(os.sched_getaffinity(0)), 32)
    refn = reference_python_rate(task, nproc, reps=5) if not args.no_cpu else None
    return {"metric": ANALYTIC_METRIC, "task": task, "value": r["value"], "unit": UNIT,
            "reference_python_1core": ref1, "reference_python_all_cores": refn,
            "steps": steps, "ms_per_step": r["ms_per_step"], "frac": r["roofline"]["frac"],
            "roofline": r["roofline"], "gpu_launches": r["gpu_launches"],
            "f64_value": r64["value"], "f64_frac": r64["roofline"]["frac"],
            "e2e": None if e2e is None else e2e["value"], "e2e_detail": e2e,
            "config": headline_config(args, world, task, steps, 1000)}


def run_b200_analytic(args, rank, world, local_rank, dist):
    """--task <analytic>: the round-1 headline (one analytic task)."""
    import torch

    from paper_2502_08844_b200 import _native

    dev = torch.device("cuda", local_rank)
    clocks = ClockSampler(local_rank).start()
    head = measure_rollout(args, args.dtype, dev, rank, world, dist, local_rank)
    clocks.stop()
    env = head["env"]
    A, O, I, esz = head["dims"]
    e2e = measure_e2e(env, args, dev, dist, A, O, I, esz, world) if args.e2e_steps > 0 else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, threads, steps, dt = cpu_rate(args.task, args.num_envs, args.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{steps} steps x {args.num_envs} worlds in {dt:.1f}s on {threads} "
                         f"threads ({cpu_model()}); oracle/oracle.c"}
    if rank == 0:
        print(json.dumps({
            "metric": ANALYTIC_METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if esz == 4 else "f64", "data": "synthetic U(-1,1) actions in HBM",
            "config": headline_config(args, world), "roofline": head["roofline"],
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": head["gpu_launches"],
            "clocks": clocks.summary(), "library": os.path.relpath(_native.LIB_PATH, ROOT)}),
            flush=True)
    env.close()


def bench_pixels(args, dev, steps=50):
    """cartpole-balance-pixels steps (env step + 64x64 render,
    brightness, luma, 3-frame stack, visual randomisation at autoreset) through
    DeviceBatchEnv, float32, 8192 worlds.  Roofline of pixel_stack_kernel:
    write-only, 64*64*3*4 B per world-step."""
    import torch

    import paper_2502_08844_b200 as dk

    n = args.num_envs
    env = dk.DeviceBatchEnv(dk.EnvConfig(task="cartpole-balance-pixels",
                                         visual_randomization=True), n, dtype="float32")
    env.reset(seed=0)
    acts = torch.rand((steps, n, 1), device=dev) * 2 - 1
    out = env._outputs((), False)
    for k in range(5):
        env.step(acts[k], out=out)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(steps):
        env.step(acts[k], out=out)
    e1.record()
    torch.cuda.synchronize(dev)
    env.check()
    ms = e0.elapsed_time(e1) / steps
    # the stack kernel alone
    pix = env._pix
    e0.record()
    for _ in range(steps):
        pix._stack()
    e1.record()
    torch.cuda.synchronize(dev)
    ks = e0.elapsed_time(e1) / steps / 1e3
    peak, src = hbm_peak()
    bytes_ws = 64 * 64 * 3 * 4
    # ppo.pixel_normalize of the step's stacks into the CNN policy's NCHW input
    from paper_2502_08844_b200.pixels import pixel_normalize

    px = out["pixels"]
    for _ in range(3):
        pixel_normalize(px)
    e0.record()
    for _ in range(steps):
        pixel_normalize(px)
    e1.record()
    torch.cuda.synchronize(dev)
    pn_s = e0.elapsed_time(e1) / steps / 1e3
    pn_bytes = 2 * bytes_ws  # the stack read once + the NCHW float32 input written once
    # a pixel-policy PPO rollout phase (ppo.collect_rollout with the reference's
    # default CNNPolicy 32@8x8/4-64@4x4/2-64@3x3 + 2x256 dense, MLPValue 5x256 on
    # the state, value normaliser), eager, T control steps
    from paper_2502_08844_b200 import ppo as P
    from paper_2502_08844_b200 import rollout as R

    class Cfg:
        unroll_length, reward_scaling, discounting = 10, 10.0, 0.995
        policy_obs_key, value_obs_key = "pixels", "state"

    torch.manual_seed(0)
    policy = R.make_cnn_policy(3, 64, 1).to(dev)
    value = R.make_value(5).to(dev)
    vn = P.DeviceRunningNormalizer(5, device=dev)
    obs = env.reset(seed=1)
    _, obs, _ = R.collect_rollout_device(env, policy, value, Cfg, obs, None, vn)
    torch.cuda.synchronize(dev)
    e0.record()
    reps = 3
    for _ in range(reps):
        _, obs, _ = R.collect_rollout_device(env, policy, value, Cfg, obs, None, vn)
    e1.record()
    torch.cuda.synchronize(dev)
    roll_s = e0.elapsed_time(e1) / 1e3 / reps
    env.close()
    pn = {"ms": pn_s * 1e3, "achieved": n * pn_bytes / pn_s / 1e9, "peak": peak, "unit": "GB/s",
          "frac": n * pn_bytes / pn_s / 1e9 / peak, "bytes_per_world": pn_bytes,
          "note": "two kernels: float64 sequential stats chains (streams the stack twice) "
                  "+ elementwise apply"}
    return {"metric": "cartpole-balance-pixels env-steps/s (step + render + 3-frame stack, "
                      "float32, 64x64)", "value": n / (ms / 1e3), "unit": "env_steps/s",
            "ms_per_step": ms, "worlds": n,
            "roofline": {"bound": "hbm", "kernel": "pixel_stack_kernel",
                         "achieved": n * bytes_ws / ks / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": n * bytes_ws / ks / 1e9 / peak, "peak_source": src,
                         "bytes_per_world_step": bytes_ws},
            "pixel_normalize": pn,
            "pixel_policy_rollout": {"value": n * Cfg.unroll_length / roll_s,
                                     "unit": "env_steps/s", "ms_per_phase": roll_s * 1e3,
                                     "phase": f"T={Cfg.unroll_length} x {n} worlds, eager, "
                                              "CNN policy float32 (cuDNN)"},
            "reference_cpu": {"value": 3.4e3, "unit": "env_steps/s",
                              "sample": "SURVEY.md §8f: BatchEnv('cartpole-balance-pixels'), "
                                        "N=256, one core"}}


def bench_ppo_rollout(args, dev, T=30, reps=5):
    """ppo.collect_rollout on the device (RolloutGraph: the
    reference's default MLPPolicy 4x128 / MLPValue 5x256, sampling, env step,
    truncation bootstrap, normalisers) + compute_gae, per phase of T control
    steps over the bench's worlds; MLPs on the tensor cores (mlp_tc_kernel,
    tcgen05 BF16x3) and, for comparison, as torch nn.Linear (cuBLAS float32).
    Reference measured in the build container: 9.7e3 env-steps/s (N=1024, 16
    torch threads)."""
    import torch

    import paper_2502_08844_b200 as dk
    from paper_2502_08844_b200 import ppo as P
    from paper_2502_08844_b200 import rollout as R

    class Cfg:
        unroll_length, reward_scaling, discounting = T, 10.0, 0.995
        policy_obs_key = value_obs_key = "state"

    n = args.num_envs
    res = {}
    for tc in (True, False):
        torch.manual_seed(0)
        env = dk.DeviceBatchEnv(dk.EnvConfig(task=args.analytic_task), n, dtype="float32")
        obs = env.reset(seed=0)
        od, ad = env.obs_dim, env.action_dim
        policy, value = R.make_policy(od, ad).cuda(dev), R.make_value(od).cuda(dev)
        pn, vn = P.DeviceRunningNormalizer(od), P.DeviceRunningNormalizer(od)
        rg = R.RolloutGraph(env, policy, value, Cfg, obs, pn, vn, tensor_cores=tc)
        for _ in range(2):
            rg.run()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            batch, _, _ = rg.run()
            P.compute_gae_batch(batch.rewards, batch.values, batch.bootstrap, batch.dones,
                                0.995, 0.95)
        e1.record()
        torch.cuda.synchronize(dev)
        env.check()
        ms = e0.elapsed_time(e1) / reps
        env.close()
        res["tensor_cores" if tc else "cublas_fp32"] = {"value": T * n / (ms / 1e3),
                                                        "ms_per_phase": ms}
    return {"metric": "env-steps/s of on-device PPO rollout collection incl. policy + value "
                      "inference (CUDA graph)", "value": res["tensor_cores"]["value"],
            "unit": "env_steps/s", "ms_per_phase": res["tensor_cores"]["ms_per_phase"],
            "cublas_fp32": res["cublas_fp32"], "unroll_length": T, "worlds": n,
            "reference_cpu": {"value": 9.7e3, "unit": "env_steps/s",
                              "sample": "ppo.collect_rollout, N=1024, T=30, 16 torch threads, "
                                        "build container (not the GPU box)"}}


def bench_go1_ppo_rollout(args, dev, T=30, reps=3):
    """The PPO rollout on the headline env: DeviceGo1Env at the bench's worlds,
    an asymmetric actor-critic of the reference's shapes (MLPPolicy on the
    56-wide noisy observation -> 12 joint means, MLPValue on the 75-wide
    privileged one) on the tensor cores, the fused step bookkeeping, truncation
    bootstraps from the terminal privileged rows; eager phases (collect_rollout_device)."""
    import torch

    from paper_2502_08844_b200 import go1env as G
    from paper_2502_08844_b200 import ppo as P
    from paper_2502_08844_b200 import rollout as R

    class Cfg:
        unroll_length, reward_scaling, discounting = T, 1.0, 0.97
        policy_obs_key, value_obs_key = "state", "privileged_state"

    n = args.num_envs
    res = {}
    for graph in (True, False):
        torch.manual_seed(0)
        env = G.DeviceGo1Env(n, G.Go1Config(), dtype="float32", device=dev.index)
        obs = env.reset(seed=0)
        pol, val = R.make_policy(56, 12).cuda(dev), R.make_value(75).cuda(dev)
        pn, vn = P.DeviceRunningNormalizer(56), P.DeviceRunningNormalizer(75)
        if graph:
            rg = R.RolloutGraph(env, pol, val, Cfg, obs, pn, vn)
            phase = lambda o: rg.run()  # noqa: E731
        else:
            phase = lambda o: R.collect_rollout_device(env, pol, val, Cfg, o, pn, vn)  # noqa: E731
        batch, obs, _ = phase(obs)
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            batch, obs, _ = phase(obs)
            P.compute_gae_batch(batch.rewards, batch.values, batch.bootstrap, batch.dones, 0.97,
                                0.95)
        b.record()
        torch.cuda.synchronize(dev)
        env.check()
        res["graph" if graph else "eager"] = a.elapsed_time(b) / reps
        env.close()
    ms = res["graph"]
    return {"metric": "env-steps/s of on-device PPO rollout collection on the Go1 joystick env "
                      "(asymmetric actor-critic on tcgen05, CUDA graph)",
            "value": T * n / (ms / 1e3), "unit": "env_steps/s", "ms_per_phase": ms,
            "physics_steps_per_s": T * n * GO1_SUBSTEPS / (ms / 1e3),
            "eager": {"value": T * n / (res["eager"] / 1e3), "ms_per_phase": res["eager"]},
            "unroll_length": T, "worlds": n}


def bench_dropin_step(args, dev, steps=300):
    """The reference-facing call itself: BatchEnv.step(numpy actions) ->
    numpy obs/rewards/dones/truncs/infos (float64, like the reference)."""
    import paper_2502_08844_b200 as dk

    env = dk.BatchEnv(dk.EnvConfig(task=args.analytic_task), args.num_envs, dtype="float64",
                      device=dev.index)
    env.reset(seed=0)
    acts = np.random.default_rng(0).uniform(-1, 1, (steps + 10, args.num_envs, env.action_dim))
    for k in range(10):
        env.step(acts[k])
    t0 = time.perf_counter()
    for k in range(steps):
        env.step(acts[10 + k])
    dt = time.perf_counter() - t0
    env.close()
    return {"value": steps * args.num_envs / dt, "unit": UNIT, "steps": steps,
            "us_per_call": dt / steps * 1e6,
            "api": "paper_2502_08844_b200.BatchEnv.step (numpy in/out, f64, infos list)"}


def bench_sweep(args, dev, sizes=(1024, 8192, 65536), K=1000, launches=5):
    """Worlds-per-GPU sweep (BASELINE config 5 style): device-resident rollout
    throughput and roofline fraction at each size."""
    import torch

    import paper_2502_08844_b200 as dk

    out = []
    peak, _ = hbm_peak()
    for n in sizes:
        env = dk.DeviceBatchEnv(dk.EnvConfig(task=args.analytic_task), n, dtype=args.dtype,
                                device=dev.index)
        env.reset(seed=0)
        tdt = env.dtype
        esz = 8 if tdt == torch.float64 else 4
        acts = torch.rand((K, n, env.action_dim), device=dev, dtype=tdt) * 2 - 1
        o = env._outputs((K,), True)
        env.rollout(acts, with_info=True, out=o)
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(launches):
            env.rollout(acts, with_info=True, out=o)
        b.record()
        torch.cuda.synchronize(dev)
        env.check()
        s_per = a.elapsed_time(b) / 1e3 / launches
        bpw = bytes_per_world_step(env.action_dim, env.obs_dim, len(env.info_keys), esz)
        rate = n * K / s_per
        out.append({"worlds": n, "value": rate, "unit": UNIT,
                    "frac": rate * bpw / 1e9 / peak})
        env.close()
        del acts, o
    return out


def bench_tasks(args, dev, K=1000, launches=5, cpu_seconds=1.0):
    """All four analytic tasks at the bench's world count,
    f32 and f64, device-resident; with each task's CPU-port rate (oracle, all
    host threads, ~1 s sample) beside it when CPU legs are enabled."""
    import torch

    import paper_2502_08844_b200 as dk

    n = args.num_envs
    peak, _ = hbm_peak()
    out = {}
    for task in ("cartpole-balance", "pendulum-swingup", "acrobot-swingup", "reacher-easy"):
        row = {}
        for dtype in ("float32", "float64"):
            env = dk.DeviceBatchEnv(dk.EnvConfig(task=task), n, dtype=dtype, device=dev.index)
            env.reset(seed=0)
            esz = 8 if env.dtype == torch.float64 else 4
            acts = torch.rand((K, n, env.action_dim), device=dev, dtype=env.dtype) * 2 - 1
            o = env._outputs((K,), True)
            env.rollout(acts, with_info=True, out=o)
            torch.cuda.synchronize(dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(launches):
                env.rollout(acts, with_info=True, out=o)
            b.record()
            torch.cuda.synchronize(dev)
            env.check()
            rate = n * K * launches / (a.elapsed_time(b) / 1e3)
            bpw = bytes_per_world_step(env.action_dim, env.obs_dim, len(env.info_keys), esz)
            row[dtype] = {"value": rate, "frac": rate * bpw / 1e9 / peak}
            env.close()
            del acts, o
        if not args.no_cpu:
            rate, threads, _, _ = cpu_rate(task, n, cpu_seconds)
            row["cpu_port"] = {"value": rate, "cores": threads}
        out[task] = row
    return {"unit": UNIT, "worlds": n, "tasks": out}


def synthetic_frames(R, J, F, dev, dtype, seed):
    """R LocomotionFrames drawn like gaitgen.random_frame (gaitgen.py:104-129),
    generated on the device (the reference is not available on the GPU box)."""
    import torch

    g = torch.Generator(device=dev)
    g.manual_seed(seed)

    def nrm(shape, s=1.0):
        return torch.randn(shape, generator=g, device=dev, dtype=torch.float64) * s

    def uni(shape, lo, hi):
        return torch.rand(shape, generator=g, device=dev, dtype=torch.float64) * (hi - lo) + lo

    q = nrm((R, 4))
    q = q / q.norm(dim=1, keepdim=True)
    f = {"base_orientation": q, "base_lin_vel": nrm((R, 3)), "base_ang_vel": nrm((R, 3)),
         "joint_pos": nrm((R, J)), "joint_vel": nrm((R, J), 2.0),
         "joint_torque": nrm((R, J), 5.0), "foot_height": uni((R, F), 0, 0.15),
         "foot_height_des": uni((R, F), 0, 0.15), "foot_vel_xy": nrm((R, F, 2), 0.5),
         "foot_contact": uni((R, F), 0, 1) < 0.5, "airtime": uni((R, F), 0, 0.8),
         "touchdown": uni((R, F), 0, 1) < 0.3, "phase": uni((R, F), -math.pi, math.pi),
         "command": nrm((R, 3), 0.5), "action": uni((R, J), -1, 1),
         "prev_action": uni((R, J), -1, 1), "joint_nominal": nrm((J,), 0.2),
         "joint_default": nrm((J,), 0.2), "done": uni((R,), 0, 1) < 0.1}
    for k, v in f.items():
        f[k] = v.to(torch.uint8) if v.dtype == torch.bool else v.to(dtype)
    return f


def bench_loco_small(args, dev, reps=50):
    """SURVEY §8a B4-B7 at Go1 shape (12 joints, 4 feet), 8192 worlds, float32,
    through the Python API (locomotion.*): device time per call with CUDA events
    around `reps` back-to-back calls.  These are one-pass elementwise kernels of a
    few hundred bytes per world: at 8192 worlds a call moves ~1-3 MB, so they are
    launch-bound (a few microseconds), not bandwidth-bound."""
    import torch

    from paper_2502_08844_b200 import locomotion as L

    n, J, F = args.num_envs, 12, 4
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    r = lambda *s: torch.rand(*s, generator=g, device=dev) * 2 - 1  # noqa: E731
    a, prev, q, qd = r(n, J), r(n, J), r(n, J), r(n, J)
    pd = L.PDParams(kp=20.0, kd=0.5, action_scale=0.3, q_default=[0.1] * J, mode="relative",
                    torque_limit=30.0)
    phi, raw, hist = r(n, F) * 3, r(n), torch.zeros(n, device=dev)
    obs = {"state": r(n, 56), "privileged_state": r(n, 75)}

    class Spec:
        def __init__(self, slot, scale, kind):
            self.slot, self.scale, self.kind = slot, scale, kind

    specs = [Spec("state", 0.05, "uniform"), Spec("state", 0.02, "gaussian")]
    key = L.NoiseKey(seed=1)
    dl = L.DelayLineBatch(n, J, 0, 3, per_step=False, dtype=torch.float32, device=dev)
    dl.reset(key)
    cases = {
        "B5 pd_batch (action_to_target + pd_torque)": (lambda: L.pd_batch(a, prev, q, qd, pd),
                                                       4 * J * 4 + 2 * J * 4),
        "B4 advance_phase_batch (+ phase_encode)": (lambda: L.advance_phase_batch(phi, 1.5, 0.02),
                                                    F * 4 + 3 * F * 4),
        "B6 progress_clip_reward_batch": (lambda: L.progress_clip_reward_batch(raw, hist), 16),
        "B7 apply_sensor_noise_batch (uniform + gaussian, 56-d state)":
            (lambda: L.apply_sensor_noise_batch(obs, specs, key), 2 * 56 * 4 + 2 * 75 * 4),
        "B7 DelayLineBatch.push_pop (12-d, delay <= 3)": (lambda: dl.push_pop(a), 2 * J * 4 * 2),
    }
    out = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for name, (fn, bpw) in cases.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize(dev)
        us = e0.elapsed_time(e1) / reps * 1e3
        # the same call captured once in a CUDA graph and replayed: device time
        # without the Python wrapper's host overhead
        gus = None
        if "DelayLine" not in name:  # (push_pop advances host-side ring bookkeeping)
            try:
                side = torch.cuda.Stream(device=dev)
                side.wait_stream(torch.cuda.current_stream(dev))
                with torch.cuda.stream(side):
                    fn()
                torch.cuda.current_stream(dev).wait_stream(side)
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    for _ in range(10):
                        fn()
                graph.replay()
                torch.cuda.synchronize(dev)
                e0.record()
                for _ in range(reps // 10):
                    graph.replay()
                e1.record()
                torch.cuda.synchronize(dev)
                gus = e0.elapsed_time(e1) / (reps // 10 * 10) * 1e3
            except Exception:  # pragma: no cover
                gus = None
        out[name] = {"us_per_call": us, "world_steps_per_s": n / (us / 1e6),
                     "graph_us_per_call": gus,
                     "graph_world_steps_per_s": None if gus is None else n / (gus / 1e6),
                     "alg_bytes_per_world": bpw,
                     "graph_achieved_GBps": None if gus is None else n * bpw / (gus / 1e6) / 1e9}
    return {"worlds": n, "dtype": "f32", "note": "device time per call through the Python API "
            "(host-bound at this size), and per call replayed from a CUDA graph (kernel-bound: "
            "a few microseconds of launch for ~0.1-8 MB of traffic)", "primitives": out}


def bench_go1_tail(args, dev, rank):
    """Go1-shape step tail (12 joints, 4 feet): rewards.total_reward (16 terms)
    + build_locomotion_observation with Philox noise, fused (SURVEY §8a B1+B2).
    One launch = K_TAIL steps x N worlds rows."""
    import torch

    from paper_2502_08844_b200 import locomotion as L

    n, J, F, K = args.num_envs, 12, 4, 100
    tdt = torch.float64 if args.dtype == "float64" else torch.float32
    esz = 8 if tdt == torch.float64 else 4
    ring = [synthetic_frames(K * n, J, F, dev, tdt, 10 + j) for j in range(3)]
    noise = L.ObservationNoise(0.05, 0.1, 0.2, 0.01, 1.5)
    cfg = L.RewardTermConfig()

    def run(j):
        return L.locomotion_tail(ring[j % len(ring)], cfg, noise=noise,
                                 key=L.NoiseKey(0, rank * n, None, j * K), num_worlds=n,
                                 check=False)

    for j in range(3):
        run(j)
    torch.cuda.synchronize(dev)
    launches = 12
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(launches)]
    stream = torch.cuda.current_stream(dev)
    for j in range(launches):
        evs[j][0].record(stream)
        run(j)
        evs[j][1].record(stream)
    torch.cuda.synchronize(dev)
    ms = [a.elapsed_time(b) for a, b in evs]
    avg_s = float(np.mean(ms)) / 1e3
    S = 9 + 3 * J + 3 + 2 * F
    P = S + F + J + 3
    in_bytes = esz * (4 + 3 + 3 + 3 * J + 2 * F + 2 * F + F + F + 3 + 2 * J) + 2 * F + 1
    out_bytes = esz * (2 + 16 + S + P)
    rows = K * n
    value = rows / avg_s
    peak, src = hbm_peak()
    achieved = rows * (in_bytes + out_bytes) / avg_s / 1e9
    res = {"metric": "Go1-shape step-tail world-steps/s (16-term reward + noisy obs), "
                     f"{n} worlds/GPU", "value": value, "unit": "world_steps/s",
           "rows_per_launch": rows, "avg_launch_ms": avg_s * 1e3,
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                        "frac": achieved / peak, "peak_source": src,
                        "bytes_per_world_step": in_bytes + out_bytes,
                        "traffic": ncu_traffic("go1_tail", args.dtype, n, K),
                        "kernel": "loco_tail_kernel"}}
    if rank == 0 and not args.no_cpu:
        res["cpu_baseline"] = cpu_tail_rate(n, J, F, args.cpu_seconds / 2)
    return res


def cpu_tail_rate(n, J, F, seconds):
    """The oracle's total_reward + build_locomotion_observation on all host
    threads over random Go1-shape frames (a bounded sample)."""
    from oracle import locomotion as olo
    from oracle.oracle import max_threads, use_all_host_threads

    use_all_host_threads()
    rng = np.random.default_rng(0)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    fr = {"base_orientation": q, "base_lin_vel": rng.normal(size=(n, 3)),
          "base_ang_vel": rng.normal(size=(n, 3)), "joint_pos": rng.normal(size=(n, J)),
          "joint_vel": rng.normal(0, 2, (n, J)), "joint_torque": rng.normal(0, 5, (n, J)),
          "foot_height": rng.uniform(0, .15, (n, F)), "foot_height_des": rng.uniform(0, .15, (n, F)),
          "foot_vel_xy": rng.normal(0, .5, (n, F, 2)), "foot_contact": rng.uniform(size=(n, F)) < .5,
          "airtime": rng.uniform(0, .8, (n, F)), "touchdown": rng.uniform(size=(n, F)) < .3,
          "phase": rng.uniform(-np.pi, np.pi, (n, F)), "command": rng.normal(0, .5, (n, 3)),
          "action": rng.uniform(-1, 1, (n, J)), "prev_action": rng.uniform(-1, 1, (n, J)),
          "joint_nominal": rng.normal(0, .2, J), "joint_default": rng.normal(0, .2, J),
          "done": rng.uniform(size=n) < .1}
    noise = [0.05, 0.1, 0.2, 0.01, 1.5]
    reps, t0 = 0, time.perf_counter()
    while True:
        olo.total_reward(fr)
        olo.loco_obs(fr, noise=noise, key=(0, 0, 0, reps))
        reps += 1
        dt = time.perf_counter() - t0
        if dt > seconds and reps >= 2:
            break
    return {"value": reps * n / dt, "unit": "world_steps/s", "cores": max_threads(),
            "kind": "port", "sample": f"{reps} x {n} Go1-shape frames in {dt:.1f}s; "
                                      "oracle/locomotion.c (rewards.total_reward + "
                                      "envkit.build_locomotion_observation restated)"}


def measure_e2e(env, args, dev, dist, A, O, I, esz, world, K=None, chunk=None):
    import ctypes

    import torch

    n = env.num_envs
    K = K or args.e2e_steps
    chunk = min(chunk or args.unroll, K)
    npdt = np.float64 if esz == 8 else np.float32

    def pinned(shape, dt):
        tdt = {np.float32: torch.float32, np.float64: torch.float64, np.uint8: torch.uint8}[dt]
        return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()

    acts = pinned((K, n, A), npdt)
    acts[:] = np.random.default_rng(7).uniform(-1, 1, (K, n, A))
    obs, rew = pinned((K, n, O), npdt), pinned((K, n), npdt)
    done, trunc, mask = pinned((K, n), np.uint8), pinned((K, n), np.uint8), pinned((K, n), np.uint8)
    term, info = pinned((K, n, O), npdt), pinned((K, n, I), npdt)
    lib = env._h._lib
    h = env._h.h

    def call(k):
        rc = lib.dk_env_rollout_host(h, k, chunk, acts.ctypes.data, obs.ctypes.data,
                                     rew.ctypes.data, done.ctypes.data, trunc.ctypes.data,
                                     term.ctypes.data, mask.ctypes.data, info.ctypes.data)
        if rc != 0:
            raise RuntimeError(f"dk_env_rollout_host failed: {rc}")

    call(min(K, 2 * chunk))  # warm-up (allocates the scratch ring)
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    call(K)
    dt = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([dt], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    nterm = int(mask.sum())
    h2d = n * A * esz
    d2h = n * (O * esz + esz + 1 + I * esz) + nterm * O * esz / K  # done/mask derived on host
    return {"value": K * n * world / dt, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "api": "dk_env_rollout_host (C ABI, pinned host buffers)",
            "steps": K, "chunk_steps": chunk}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test hooks for the multi-rank path on a 1-GPU box: every rank on GPU 0
    # (the ranks' kernels never wait on each other) and a gloo process group
    if os.environ.get("DK_BENCH_SAME_DEVICE") == "1":
        local_rank = 0
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(local_rank)
        backend = os.environ.get("DK_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            # communicator set-up lines on stderr (the JSON line is on stdout): the
            # transport NCCL picked (NVLink / NVLS) is in the driver's logs
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            tdist.init_process_group(backend)
        dist = tdist
    try:
        run_b200(args, rank, world, local_rank, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
