"""Build libattn2d_sm100.so in-tree with nvcc for sm_100a.

    python -m paper_2406_18485_b200.build [--force] [-v]

Objects go to ``build/``; the shared library to
``paper_2406_18485_b200/lib/libattn2d_sm100.so`` (git-ignored, but shipped to
the GPU box by gpurun's snapshot). Rebuilds only when a source or header is
newer than the library.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "lib", "libattn2d_sm100.so")
SOURCES = ["fa_fwd.cu", "fa_bwd.cu", "aux.cu", "umma_selftest.cu", "capi.cu", "runtime.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--use_fast_math", "-Xcompiler", "-fPIC",
         "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found (CUDA 12.9 toolkit required)")


def nccl_dirs() -> tuple[str, str]:
    """(include, lib) of the NCCL torch loads (2.28.x from the nvidia-nccl wheel):
    the library links and rpaths it, so whichever of torch / this library is
    loaded first, one NCCL ends up in the process (the system 2.27 would shadow
    symbols torch needs)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia.nccl (torch's NCCL wheel) not found")
    base = list(spec.submodule_search_locations)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _deps() -> list[str]:
    out = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    out.append(os.path.join(ROOT, "include", "attn2d_sm100.h"))
    return out


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force: bool = False, verbose: bool = False, profile: bool = False, variant: str = "") -> str:
    """profile=True: a separate lib/libattn2d_sm100_prof.so with -DA2D_PROFILE
    (per-role barrier wait counters in the backward, a2d_prof_read); never
    loaded by default. variant="X": also -DA2D_X, library suffix _prof_x
    (experiments, e.g. SPIN)."""
    tag = "_prof" + (f"_{variant.lower()}" if variant else "")
    lib_out = LIB.replace(".so", f"{tag}.so") if profile else LIB
    if not profile and not force and not needs_build():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    cc = nvcc()
    nccl_inc, nccl_lib = nccl_dirs()
    procs = []
    objs = []
    for src in SOURCES:
        obj = os.path.join(BUILD, src.replace(".cu", f"{tag}.o" if profile else ".o"))
        objs.append(obj)
        defs = (["-DA2D_PROFILE"] + ([f"-DA2D_{variant}"] if variant else [])) if profile else []
        cmd = [cc, *ARCH, *FLAGS, *defs, "-I", os.path.join(ROOT, "include"),
               "-I", nccl_inc, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        log = os.path.join(BUILD, src + (tag if profile else "") + ".log")
        with open(log, "w") as f:
            f.write(out)
        if verbose:
            print(f"== {src}\n{out}")
        if p.returncode != 0:
            failed.append((src, out))
    if failed:
        msg = "\n".join(f"--- {s}\n{o[-6000:]}" for s, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    tmp = lib_out + ".tmp"
    cmd = [cc, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fPIC", "-L", nccl_lib, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath={nccl_lib}"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}")
    os.replace(tmp, lib_out)
    return lib_out


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--profile", action="store_true", help="build the instrumented lib/libattn2d_sm100_prof.so")
    ap.add_argument("--variant", default="", help="with --profile: extra -DA2D_<VARIANT> (library _prof_<variant>)")
    a = ap.parse_args(argv)
    print(build(force=a.force, verbose=a.verbose, profile=a.profile, variant=a.variant))
    return 0


if __name__ == "__main__":
    sys.exit(main())
