"""Build libcurvopt_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2603_25976_b200.build      (or via __graft_entry__.build())
"""

from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIB_DIR, "libcurvopt_b200.so")
ROOT = os.path.dirname(HERE)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    try:
        import nvidia.nccl as _n  # type: ignore

        base = list(_n.__path__)[0]
        return os.path.join(base, "include"), os.path.join(base, "lib", "libnccl.so.2")
    except Exception:  # pragma: no cover
        return None, None


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _fingerprint(srcs):
    h = hashlib.sha256()
    deps = srcs + sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")))
    deps.append(os.path.join(ROOT, "include", "curvopt_b200.h"))
    deps.append(os.path.abspath(__file__))
    for p in deps:
        with open(p, "rb") as f:
            h.update(p.encode())
            h.update(f.read())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    srcs = _sources()
    os.makedirs(LIB_DIR, exist_ok=True)
    stamp = LIB + ".sha"
    fp = _fingerprint(srcs)
    if not force and os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == fp:
        return LIB
    inc, nccl_lib = _nccl_dirs()
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
                    "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
    if inc:
        flags += ["-I", inc]
    if nccl_lib:
        flags += [f'-DCV_NCCL_LIB_PATH="{nccl_lib}"']
    if os.environ.get("CURVOPT_PTXAS_V"):
        flags += ["-Xptxas", "-v"]
    build_dir = os.path.join(HERE, "build")
    os.makedirs(build_dir, exist_ok=True)
    objs = []
    procs = []
    for s in srcs:
        o = os.path.join(build_dir, os.path.basename(s) + ".o")
        objs.append(o)
        cmd = ["nvcc", *flags, "-c", s, "-o", o]
        if verbose:
            print(" ".join(cmd))
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append((cmd, out.decode()))
        elif verbose and out:
            print(out.decode())
    if failed:
        for cmd, out in failed:
            sys.stderr.write(" ".join(cmd) + "\n" + out + "\n")
        raise RuntimeError("nvcc failed")
    link = ["nvcc", *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-ldl"]
    subprocess.run(link, check=True)
    with open(stamp, "w") as f:
        f.write(fp)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
