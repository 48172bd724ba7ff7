"""Build the B200 env-step library (sm_100a) in-tree.

    python -m paper_2502_08844_b200.build

Produces paper_2502_08844_b200/libdeskrl_b200.so from csrc/*.cu with nvcc.
The float64 translation unit is compiled with --fmad=false so its arithmetic
rounds like the reference's Python floats (no fused multiply-add).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libdeskrl_b200.so")
OBJDIR = os.path.join(ROOT, "build", "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# DK_NVCC_EXTRA / DK_LIB_OUT / DK_OBJ_DIR: developer hooks for experimental
# variants (tools/exp_variants.sh); unset for the product build.
if os.environ.get("DK_LIB_OUT"):
    LIB = os.path.abspath(os.environ["DK_LIB_OUT"])
if os.environ.get("DK_OBJ_DIR"):
    OBJDIR = os.path.abspath(os.environ["DK_OBJ_DIR"])
COMMON = [*os.environ.get("DK_NVCC_EXTRA", "").split(), "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-I", os.path.join(ROOT, "include")]
UNITS = {
    "envstep_f32.cu": [],
    "envstep_f64.cu": ["--fmad=false"],
    "locomotion_f32.cu": [],
    "locomotion_f64.cu": ["--fmad=false"],
    "capi.cu": [],
    "capi_loco.cu": [],
    "capi_ppo.cu": ["--fmad=false"],
    "capi_pixels.cu": ["--fmad=false"],
    # float32 physics / Go1 env: division and sqrt through MUFU reciprocal /
    # square-root approximations (<= 2 ulp), FTZ.  +5% on the Go1 env with the
    # physics parity report unchanged (100-step divergence fractions equal;
    # --use_fast_math was +11% but its __sinf / __expf made 4x more worlds
    # diverge past 1e-3 at 100 steps -- rejected).
    "physics_f32.cu": ["-prec-div=false", "-prec-sqrt=false", "-ftz=true"],
    "physics_f64.cu": ["--fmad=false"],
    "capi_phys.cu": [],
    "go1env_f32.cu": ["-prec-div=false", "-prec-sqrt=false", "-ftz=true"],
    "go1env_f64.cu": ["--fmad=false"],
    "capi_go1.cu": [],
    "capi_mlp.cu": [],
}


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a env-step library")


def _sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
            if f.endswith((".cu", ".cuh", ".h"))] + [os.path.join(ROOT, "include", "deskrl_b200.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nvcc = _nvcc()
    os.makedirs(OBJDIR, exist_ok=True)
    objs, cmds = [], []
    for unit, extra in UNITS.items():
        obj = os.path.join(OBJDIR, unit.replace(".cu", ".o"))
        cmds.append([nvcc, *ARCH, *COMMON, *extra, "-Xptxas", "-v" if verbose else "-O3", "-c",
                     os.path.join(CSRC, unit), "-o", obj])
        objs.append(obj)
    # translation units are independent: compile them concurrently
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        for r in list(ex.map(lambda c: subprocess.run(c, check=True), cmds)):
            pass
    tmp = LIB + ".tmp"
    subprocess.run([nvcc, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
