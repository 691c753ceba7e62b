"""Build libwos_b200.so in-tree with nvcc for sm_100a (no GPU needed).

    python -m paper_2603_01193_b200.build [--force] [--jobs N]

Each numeric mode is its own translation unit so the REPLAY units can be
compiled without FMA contraction (--fmad=false: the reference's numpy/numba
arithmetic never fuses multiply-add), while the NATIVE unit keeps FFMA.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libwos_b200.so")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--expt-relaxed-constexpr", "-I", os.path.join(HERE, "..", "include"),
]
UNITS = {
    "wos_capi.cu": [],
    "wos_kernels_native.cu": [],
    "wos_kernels_native_est.cu": [],
    # the 10-round hot kernels (cfg4, cfg0) run two walks per lane at 3 CTAs/SM (80
    # registers): -2 to -3 % against one walk at 4 CTAs/SM; the 7-round ones do not
    # gain from it (round 2). (7-warp CTAs at 4 CTAs/SM, -DWOS_NW=7:
    # 28 resident warps at 72 registers, were 1.7 % slower on cfg4)
    "wos_kernels_native_est_bc.cu": ["-DWOS_ILP2=1", "-DWOS_NATIVE_MINB=3"],
    "wos_kernels_native_est_r7.cu": [],
    "wos_kernels_native_est_bc_r7.cu": [],
    "wos_kernels_native_rows.cu": [],
    "wos_kernels_replay_f64.cu": ["--fmad=false"],
    "wos_kernels_replay_f32.cu": ["--fmad=false"],
    "wos_cache.cu": ["--fmad=false"],
}
HEADERS = ["wos_types.h", "wos_rng.cuh", "wos_walk.cuh", "wos_mesh.cuh", "wos_kernels.h",
           "wos_kernels_native.inc"]


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, extra, verbose, build_dir=None):
    obj = os.path.join(build_dir or BUILD, src.replace(".cu", ".o"))
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(HERE, "..", "include", "wos_b200.h")
    ]
    if not _stale(obj, deps):
        return obj, None
    cmd = [NVCC] + COMMON + extra + ["-Xptxas", "-v", "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    with open(obj + ".ptxas.txt", "w") as fh:
        fh.write(r.stderr)
    return obj, r.stderr if verbose else None


def build(force: bool = False, jobs: int | None = None, verbose: bool = False, defines=(),
          out: str | None = None) -> str:
    """Compile every unit and link the shared library.

    ``defines``/``out`` build an experimental variant (e.g. WOS_NATIVE_MINB=3) into a
    separate directory and library; load it with WOS_B200_LIB=<path>.
    """
    build_dir = BUILD if not out else os.path.join(HERE, "_build_" + os.path.basename(out).split(".")[0])
    lib = LIB if not out else os.path.join(HERE, out)
    os.makedirs(build_dir, exist_ok=True)
    if force:
        for f in os.listdir(build_dir):
            os.remove(os.path.join(build_dir, f))
    extra_d = [f"-D{d}" for d in defines]
    jobs = jobs or min(len(UNITS), os.cpu_count() or 1)
    with cf.ThreadPoolExecutor(jobs) as ex:
        futs = [ex.submit(_compile, s, e + extra_d, verbose, build_dir) for s, e in UNITS.items()]
        objs = []
        for f in futs:
            obj, log = f.result()
            objs.append(obj)
            if log:
                print(log, file=sys.stderr)
    if force or _stale(lib, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    print(build(a.force, a.jobs, a.verbose, a.defines, a.out))
