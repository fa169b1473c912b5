"""Build the in-tree CUDA extension libsbattn.so (sm_100a only).

Plain nvcc, no torch build machinery: the library exports the C ABI declared in
include/sb_attn.h and is loaded with ctypes.  `python -m paper_2410_17980_b200.build`
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsbattn.so")
SOURCES = ["sb_api.cu", "sb_fwd_pp.cu", "sb_bwd.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"),
]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "sb_attn.h"))
    return any(os.path.getmtime(d) > t for d in deps)


LIB_TRACE = os.path.join(HERE, "libsbattn_trace.so")


def build(force: bool = False, verbose: bool = False, trace: bool = False,
          variant: str = "", defines: tuple = ()) -> str:
    """Compile libsbattn.so (or, with trace=True, the -DSB_TRACE tuning variant
    libsbattn_trace.so that records per-event SM clocks, tools/trace_kernels.py;
    variant="nomath" builds libsbattn_nomath.so, the pipeline without the stick
    math, for tools/ablate.py)."""
    lib = LIB_TRACE if trace else LIB
    tag = "_trace" if trace else ""
    extra = ["-DSB_TRACE"] if trace else []
    if variant:
        lib = os.path.join(HERE, f"libsbattn_{variant}.so")
        tag = "_" + variant
        extra = {"nomath": ["-DSB_NOMATH"], "trace_nomath": ["-DSB_NOMATH", "-DSB_TRACE"],
                 "noz": ["-DSB_NOZ"], "nomath_noz": ["-DSB_NOMATH", "-DSB_NOZ"]}.get(variant, [])
        extra = extra + ["-D" + d for d in defines]  # tuning A/B builds (tools/ablate.py)
    if not force and not _stale(lib):
        return lib
    jobs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        if not os.path.exists(path):
            continue
        # per-process object names and an atomic rename of the library: several ranks
        # (torchrun) may find the library stale at once
        obj = os.path.join(CSRC, src.replace(".cu", f"{tag}.{os.getpid()}.o"))
        cmd = [NVCC, *FLAGS, *extra, "-c", path, "-o", obj]
        jobs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                stderr=subprocess.STDOUT, text=True)))
    objs, log = [], []
    for src, obj, proc in jobs:
        out = proc.communicate()[0]
        log.append(out)
        if proc.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{out}")
        objs.append(obj)
    tmp = f"{lib}.{os.getpid()}.tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
           "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    for o in objs:
        os.remove(o)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    if verbose:
        print("\n".join(log))
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv))
