"""Build the sm_100a CUDA library in-tree (nvcc cross-compiles without a GPU).

    python -m paper_2502_08910_b200.build
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "_lib"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
              f"-I{ROOT / 'include'}", f"-I{CSRC}"]
CUDA_SOURCES = ["prune.cu", "bsa.cu", "decode.cu", "layer.cu", "cache.cu", "prefill.cu", "capi.cu"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build_cuda(force: bool = False, verbose: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    # dev builds: HP_TRACE=1 -> phase cuts + per-CTA phase tracer; HP_TRACE=cuts -> cuts only
    traced = os.environ.get("HP_TRACE") in ("1", "cuts")
    dev_flags = (["-DHP_TRACE"] + (["-DHP_CUTS_ONLY"] if os.environ.get("HP_TRACE") == "cuts" else [])) if traced else []
    out = LIB / ("libhipprune_b200_trace.so" if traced else "libhipprune_b200.so")
    # dev A/B builds: HP_VARIANT=name HP_VARIANT_FLAGS="-DX=1" -> _lib/libhipprune_b200_<name>.so
    variant = os.environ.get("HP_VARIANT")
    if variant:
        out = LIB / f"libhipprune_b200_{variant}.so"
        dev_flags = dev_flags + ["-DHP_DEV"] + os.environ.get("HP_VARIANT_FLAGS", "").split()
    deps = [CSRC / s for s in CUDA_SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "hipprune_b200.h"]
    if not force and not _stale(out, deps):
        return out
    objs, procs = [], []
    for src in CUDA_SOURCES:  # compile translation units in parallel
        obj = LIB / (Path(src).stem + (f".{variant}" if variant else "") + (".trace.o" if traced else ".o"))
        cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *dev_flags, "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd)))
        objs.append(str(obj))
    for src, p in procs:
        if p.wait() != 0:
            raise RuntimeError(f"nvcc failed on {src}")
    subprocess.run([nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", str(out)], check=True)
    for o in objs:
        Path(o).unlink(missing_ok=True)
    return out


HOST_SOURCES = ["host/host.cpp", "host/decode_engine.cpp", "host/kv_store.cpp"]


def _cuda_home() -> Path:
    return Path(nvcc()).resolve().parent.parent


def build_host(force: bool = False) -> Path:
    """The C++ host layer (include/hipprune_b200.hpp) over the C ABI, and the
    reference-named pybind11 module _hipprune on top of it."""
    import sysconfig
    import pybind11
    cuda = _cuda_home()
    cxx = os.environ.get("CXX", "g++")
    host = LIB / "libhipprune_host.so"
    deps = [CSRC / s for s in HOST_SOURCES] + list((ROOT / "include" / "hipprune").glob("*.hpp")) + [ROOT / "include" / "hipprune_b200.hpp",
                                             ROOT / "include" / "hipprune_b200.h", LIB / "libhipprune_b200.so"]
    common = ["-O2", "-std=c++20", "-fPIC", "-ffp-contract=off", f"-I{ROOT / 'include'}", f"-I{cuda / 'include'}"]
    links = [f"-L{LIB}", "-lhipprune_b200", f"-L{cuda / 'lib64'}", "-lcudart", "-lz", "-Wl,-rpath,$ORIGIN",
             f"-Wl,-rpath,{cuda / 'lib64'}"]
    if force or _stale(host, deps):
        subprocess.run([cxx, *common, "-shared", *[str(CSRC / s) for s in HOST_SOURCES], "-o", str(host), *links],
                       check=True)
    ext = LIB / ("_hipprune" + sysconfig.get_config_var("EXT_SUFFIX"))
    bdeps = [CSRC / "host" / "bindings.cpp", host]
    if force or _stale(ext, bdeps):
        subprocess.run([cxx, *common, "-shared", f"-I{pybind11.get_include()}",
                        f"-I{sysconfig.get_paths()['include']}", str(CSRC / "host" / "bindings.cpp"), "-o", str(ext),
                        f"-L{LIB}", "-lhipprune_host", *links], check=True)
    return ext


def build(force: bool = False) -> None:
    build_cuda(force=force)
    if os.environ.get("HP_TRACE") not in ("1", "cuts"):
        build_host(force=force)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print("built", LIB)
