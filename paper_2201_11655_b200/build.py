"""Compile libvdmc.so for sm_100a with nvcc (in-tree, so it travels with the repo).
The translation units compile in parallel (one nvcc per .cu), then link into one .so."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libvdmc.so")
SOURCES = ["api.cu", "build.cu", "enum.cu", "enum32.cu", "edges.cu", "layers.cu"]

def _nccl_dir() -> str:
    """NCCL 2.28 as shipped with torch (nvidia-nccl wheel): headers and libnccl.so.2."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia.nccl (NCCL headers + libnccl.so.2) not found")
    return list(spec.submodule_search_locations)[0]


NCCL = _nccl_dir()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-I", os.path.join(NCCL, "include")]
LINK = ["-L" + os.path.join(NCCL, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib")]


def build(force: bool = False, verbose: bool = False, lib: str = LIB, defines=()) -> str:
    """Compile and link libvdmc.so.  defines=("VDMC_PROFILING",) gives the profiling variant
    (tools/ only: switches that drop work for phase timings)."""
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "vdmc_internal.cuh"), os.path.join(CSRC, "enum.cu"),
                   os.path.join(HERE, "..", "include", "vdmc.h")]
    if not force and os.path.exists(lib) and \
            os.path.getmtime(lib) >= max(os.path.getmtime(d) for d in deps):
        return lib
    os.makedirs(LIBDIR, exist_ok=True)
    tag = f".tmp{os.getpid()}"
    objs = [os.path.join(LIBDIR, os.path.basename(s) + tag + ".o") for s in srcs]
    dflags = [f"-D{d}" for d in defines]
    procs = [subprocess.Popen(["nvcc", *FLAGS, *dflags, "-c", "-o", o, s], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for s, o in zip(srcs, objs)]
    logs, ok = [], True
    for p in procs:
        out, err = p.communicate()
        logs.append(out + err)
        ok &= p.returncode == 0
    try:
        if not ok:
            sys.stderr.write("".join(logs))
            raise RuntimeError("nvcc failed building libvdmc.so")
        tmp = lib + tag
        res = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, *LINK],
                             capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed linking libvdmc.so")
        if verbose:
            sys.stderr.write("".join(logs))
        os.replace(tmp, lib)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.unlink(o)
    return lib


def build_profiling(force: bool = False) -> str:
    """libvdmc_prof.so: the same sources with -DVDMC_PROFILING (tools/phase_probe.py)."""
    return build(force=force, lib=os.path.join(LIBDIR, "libvdmc_prof.so"), defines=("VDMC_PROFILING",))


if __name__ == "__main__":
    print(build(force=True, verbose=True))
