"""Compile libvdmc.so for sm_100a with nvcc (in-tree, so it travels with the repo).
The translation units compile in parallel (one nvcc per .cu), then link into one .so."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libvdmc.so")
SOURCES = ["api.cu", "build.cu", "enum.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "vdmc_internal.cuh"),
                   os.path.join(HERE, "..", "include", "vdmc.h")]
    if not force and os.path.exists(LIB) and \
            os.path.getmtime(LIB) >= max(os.path.getmtime(d) for d in deps):
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    tag = f".tmp{os.getpid()}"
    objs = [os.path.join(LIBDIR, os.path.basename(s) + tag + ".o") for s in srcs]
    procs = [subprocess.Popen(["nvcc", *FLAGS, "-c", "-o", o, s], stdout=subprocess.PIPE,
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
        tmp = LIB + tag
        res = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs],
                             capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed linking libvdmc.so")
        if verbose:
            sys.stderr.write("".join(logs))
        os.replace(tmp, LIB)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.unlink(o)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
