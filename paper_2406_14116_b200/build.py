"""In-tree build of the CUDA extension ``libfcvbw_gpu.so`` (sm_100a) with nvcc.

The translation units are compiled in parallel (the fp32 and fp64 kernel instantiations dominate),
then linked into one shared library with the CUDA runtime linked statically, so the .so that
travels to the GPU box has no dependency on a JIT cache or on torch.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libfcvbw_gpu.so")
SOURCES = ["fcvbw_gpu.cu", "kernels_f32.cu", "kernels_f64.cu", "kernels_f32_real.cu", "kernels_f64_real.cu", "kernels_f32_dump.cu", "kernels_f64_dump.cu", "verify.cu", "design.cu", "analyze.cu", "workload.cu"]
HEADERS = ["cplx.cuh", "dft.cuh", "launch.cuh", "ols_kernel.cuh", "kernels_impl.cuh", "twiddle64.cuh", "sm100.cuh",
           "grid.h", "response.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA extension cannot be built")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, lib: str = LIB, build_dir: str = BUILD,
          defines: tuple = ()) -> str:
    os.makedirs(build_dir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(HERE, "..", "include", "fcvbw_gpu.h")]
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return r

    with cf.ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(lib, objs):
        run([nvcc(), *ARCH, "-shared", "-o", lib, *objs, "-cudart", "static"])
    return lib


if __name__ == "__main__":
    # experiment variants: python build.py --variant NAME -DFOO=1 ... -> _variants/NAME/libfcvbw_gpu.so
    if "--variant" in sys.argv:
        name = sys.argv[sys.argv.index("--variant") + 1]
        defs = tuple(a[2:] for a in sys.argv if a.startswith("-D"))
        d = os.path.join(HERE, "_variants", name)
        print(build(force=True, lib=os.path.join(d, "libfcvbw_gpu.so"), build_dir=d, defines=defs))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
