"""Build the C-ABI shared library ``libkx.so`` in-tree (nvcc, sm_100a).

    python -m paper_2310_07551_b200.build        # or __graft_entry__.build()

Every translation unit under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked with the static CUDA
runtime into paper_2310_07551_b200/libkx.so.  Rebuilds only when a source is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OUT = os.path.join(PKG, "libkx.so")
BUILD = os.path.join(ROOT, "build", "kx")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC]


def nccl_include() -> str | None:
    """nccl.h of the NCCL that torch loads (pip wheel nvidia-nccl-cu12), so the process has a
    single NCCL; the library dlopens libnccl.so.2 at kx_create_dist time."""
    try:
        import nvidia.nccl as m
        for base in list(getattr(m, "__path__", [])):
            inc = os.path.join(base, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except Exception:
        pass
    return None


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cpp")))


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(dp) > t for dp in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".h")]
    headers.append(os.path.join(INCLUDE, "kx.h"))
    objs, jobs = [], []
    for src in sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _newer(obj, [src] + headers):
            cmd = [nvcc()] + ARCH + COMMON
            inc = nccl_include()
            if inc:
                cmd += ["-I", inc, "-DKX_HAVE_NCCL"]
            if src.endswith(".cu") and verbose:
                cmd += ["-Xptxas", "-v"]
            cmd += ["-c", src, "-o", obj]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for err in ex.map(run, jobs):
            if verbose and err:
                sys.stderr.write(err)
    if force or jobs or _newer(OUT, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", OUT] + objs + ["-cudart", "static", "-ldl"]
        run(cmd)
    build_examples()
    build_tools()
    return OUT


def build_tools() -> None:
    """Standalone CUDA microbenchmarks (tools/*.cu, e.g. the fp64 DMMA / DFMA / HBM peaks that
    bench.py measures in the same job) -> build/<name>.  Not part of the product path."""
    tdir = os.path.join(ROOT, "tools")
    if not os.path.isdir(tdir):
        return
    for f in sorted(os.listdir(tdir)):
        if not f.endswith(".cu"):
            continue
        src = os.path.join(tdir, f)
        exe = os.path.join(ROOT, "build", f[:-3])
        if not _newer(exe, [src]):
            continue
        cmd = [nvcc()] + ARCH + ["-O3", "-std=c++17", "-lineinfo", "-o", exe, src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"tool build failed: {' '.join(cmd)}\n{r.stderr}")


def build_examples() -> None:
    """C clients of the ABI (examples/*.c) -> build/<name>, linked against libkx.so."""
    ex_dir = os.path.join(ROOT, "examples")
    cc = shutil.which("gcc")
    if not cc or not os.path.isdir(ex_dir):
        return
    cuda = os.path.dirname(os.path.dirname(nvcc()))
    for f in sorted(os.listdir(ex_dir)):
        if not f.endswith(".c"):
            continue
        src = os.path.join(ex_dir, f)
        exe = os.path.join(ROOT, "build", f[:-2])
        if not _newer(exe, [src, OUT, os.path.join(INCLUDE, "kx.h")]):
            continue
        cmd = [cc, "-O2", "-o", exe, src, "-I", INCLUDE, "-I", os.path.join(cuda, "include"),
               "-L", PKG, "-lkx", "-L", os.path.join(cuda, "lib64"), "-lcudart",
               "-Wl,-rpath," + PKG]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"example build failed: {' '.join(cmd)}\n{r.stderr}")


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
