"""Build libedl.so (the C-ABI library) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libedl.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources(logns=None):
    """All .cu/.cpp sources; `logns` (development builds) keeps only those ring degrees'
    ntt_inst_<logN>.cu instantiation units."""
    out = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    if logns:
        keep = {f"ntt_inst_{k}.cu" for k in logns}
        out = [p for p in out if not os.path.basename(p).startswith("ntt_inst_") or os.path.basename(p) in keep]
    return out


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        [os.path.join(os.path.dirname(HERE), "include", "edl.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None, logns=None) -> str:
    lib = out or LIB
    if logns:
        assert out is not None, "a trimmed build must not replace the product library"
        defines = tuple(defines) + (f"EDL_LOGNS_MASK={sum(1 << k for k in logns)}",)
    if not force and not defines and out is None and up_to_date():
        return LIB
    objdir = os.path.join(HERE, "build" + ("_" + "_".join(d.replace("=", "") for d in defines) if defines else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    hdr_time = max(os.path.getmtime(p) for p in deps() if not p.endswith((".cu", ".cpp")))
    for src in sources(logns):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(hdr_time, os.path.getmtime(src)):
            objs.append(obj)    # incremental: object newer than its source and every header
            continue
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
               "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3",
               *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    ok = True
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out.decode())
        ok &= p.returncode == 0
    if not ok:
        raise RuntimeError("nvcc failed")
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    ln = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--logns=")]
    logns = [int(x) for x in ln[0].split(",")] if ln else None
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, out=outs[0] if outs else None,
                logns=logns))
