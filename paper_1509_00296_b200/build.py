"""Build libfrsvt.so in-tree for sm_100a (B200). No GPU needed: nvcc
cross-compiles. Used by __graft_entry__.build() and by hand:

    python paper_1509_00296_b200/build.py [--force] [-v]

(run as a script or through __graft_entry__.build(): importing the package
loads libfrsvt.so, so the builder must not import it)
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libfrsvt.so")
SOURCES = [os.path.join(HERE, "csrc", "frsvt.cu")]


def _nccl_dirs():
    import nvidia.nccl  # torch's NCCL (same library torch.distributed loads)
    base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc_cmd(out=LIB, extra=()):
    inc, lib = _nccl_dirs()
    return ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
            "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v",
            "-I", os.path.join(ROOT, "include"), "-I", os.path.join(HERE, "csrc"), "-I", inc,
            *SOURCES, "-o", out, "-L", lib, "-l:libnccl.so.2", "-ldl", "-Xlinker", "-rpath=" + lib,
            *extra]


STAMP = LIB + ".sha256"


def source_digest():
    """sha256 over the library's sources and the compile command: a prebuilt
    .so is reused only if it was built from exactly these bytes."""
    import hashlib
    hsh = hashlib.sha256()
    deps = [os.path.join(ROOT, "include", "frsvt.h")]
    csrc = os.path.join(HERE, "csrc")
    deps += sorted(os.path.join(csrc, f) for f in os.listdir(csrc) if f.endswith((".cu", ".cuh", ".h")))
    for p in deps:
        hsh.update(os.path.relpath(p, ROOT).encode())
        with open(p, "rb") as f:
            hsh.update(f.read())
    hsh.update(" ".join(nvcc_cmd()[:12]).encode())
    return hsh.hexdigest()


def needs_build():
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    with open(STAMP) as f:
        return f.read().strip() != source_digest()


def build(force=False, verbose=False):
    if not force and not needs_build():
        return LIB
    digest = source_digest()
    cmd = nvcc_cmd()
    p = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
    if p.returncode != 0:
        sys.stderr.write(p.stderr[-8000:])
        raise RuntimeError("nvcc failed building libfrsvt.so (see %s)" % log)
    if verbose:
        sys.stderr.write(p.stderr)
    with open(STAMP, "w") as f:
        f.write(digest + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
