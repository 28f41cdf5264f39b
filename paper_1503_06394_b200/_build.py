"""Build libchebld.so in-tree with nvcc for sm_100a (called by __graft_entry__.build())."""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libchebld.so")
SOURCES = [os.path.join(CSRC, "cheb_logdet.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "cheb_kernels.cuh"), os.path.join(ROOT, "include", "cheb_logdet.h")]

NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile libchebld.so (or a tuning variant at `out` with extra -D defines)."""
    so = out or SO
    if not force and os.path.exists(so) and all(os.path.getmtime(so) >= os.path.getmtime(d) for d in DEPS):
        return so
    tmp = so + f".tmp{os.getpid()}"
    cmd = [nvcc()] + NVCC_FLAGS + [f"-D{d}" for d in defines] + ["-I", os.path.join(ROOT, "include"), "-o", tmp] + SOURCES
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(CSRC, "ptxas.log" if out is None else "ptxas_" + os.path.basename(so) + ".log")
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed: " + " ".join(cmd))
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, so)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
