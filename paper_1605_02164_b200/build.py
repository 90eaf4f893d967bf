"""Build libbfvec.so (the C-ABI library) in-tree for sm_100a.

    python paper_1605_02164_b200/build.py [--force]

Each .cu under csrc/ is compiled by nvcc in parallel, then linked into
paper_1605_02164_b200/libbfvec.so (static CUDA runtime). ptxas resource usage
(-Xptxas -v) is written to build/ptxas_<file>.log.
"""
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# A/B experiments: BFVEC_BUILD_TAG=x builds build/obj_x -> libbfvec_x.so with the extra nvcc flags
# in BFVEC_NVCC_EXTRA (e.g. -DBFVEC_MBAR_SPIN); load it with BFVEC_LIB=<path> (_lib.py)
TAG = os.environ.get("BFVEC_BUILD_TAG", "")
OBJ = os.path.join(ROOT, "build", "obj" + (f"_{TAG}" if TAG else ""))
LIB = os.path.join(HERE, f"libbfvec{'_' + TAG if TAG else ''}.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"),
         *os.environ.get("BFVEC_NVCC_EXTRA", "").split()]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps_mtime(src):
    """Newest mtime of src and every local header it includes (transitively)."""
    seen, todo = set(), [os.path.join(CSRC, src)]
    while todo:
        f = todo.pop()
        if f in seen or not os.path.exists(f):
            continue
        seen.add(f)
        for line in open(f, encoding="utf-8", errors="replace"):
            line = line.strip()
            if line.startswith("#include \""):
                name = line.split('"')[1]
                todo.append(os.path.normpath(os.path.join(os.path.dirname(f), name)))
    return max(os.path.getmtime(f) for f in seen)


def _compile(src, force):
    obj = os.path.join(OBJ, src.replace(".cu", ".o"))
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= _deps_mtime(src):
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = res.stdout + res.stderr
    with open(os.path.join(ROOT, "build", f"ptxas_{src}{'_' + TAG if TAG else ''}.log"), "w") as fh:
        fh.write(log)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{log[-6000:]}")
    return obj, log


def build(force: bool = False, jobs: int = 0) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = [o for o, _ in ex.map(lambda s: _compile(s, force), srcs)]
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("link failed:\n" + res.stdout + res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
