"""Builds libtm.so (the C-ABI library, include/tm.h) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import json
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libtm.so")
STAMP = LIB + ".build.json"  # source hash + the exact nvcc commands of the build that produced LIB
SOURCES = ["api.cpp", "plan.cpp", "dist.cpp", "tune.cpp", "simt_gemm.cu", "small_gemm.cu", "tc_gemm_nn.cu", "tc_gemm_nt.cu", "tc_gemm_tn.cu", "tc_gemm_tt.cu", "tc_conv.cu", "tc_conv_direct.cu", "blur.cu", "ce_chain.cpp"]
HEADERS = ["ptx.cuh", "tm_internal.h", "tc_gemm.cuh"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "--expt-relaxed-constexpr", f"-I{os.path.join(ROOT, 'include')}"]


def _source_hash(extra: list[str]) -> str:
    """sha256 over every source, header, this build script and the flags: a
    library is reused only if it was built from exactly these bytes (mtimes of a
    copied tree prove nothing)."""
    h = hashlib.sha256()
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "tm.h"), __file__]
    for d in deps:
        h.update(os.path.basename(d).encode())
        with open(d, "rb") as f:
            h.update(f.read())
    h.update(" ".join([NVCC, *ARCH, *FLAGS, *extra]).encode())
    return h.hexdigest()


def _stale(extra: list[str]) -> bool:
    if not (os.path.exists(LIB) and os.path.exists(STAMP)):
        return True
    try:
        with open(STAMP) as f:
            return json.load(f).get("source_sha256") != _source_hash(extra)
    except (OSError, ValueError):
        return True


def _compile(src: str, extra: list[str], obj_dir: str) -> tuple[str, list[str]]:
    obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    if src.endswith(".cpp"):
        cmd[cmd.index("-c"):cmd.index("-c")] = ["-x", "cu"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj, cmd


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None, out: str | None = None) -> str:
    """Compile every source into a fresh object directory and link libtm.so,
    unless the library's stamp records a build from exactly these sources and
    flags (force=True always rebuilds).  The stamp lists the nvcc commands.
    out: another library path (tests' mutant builds, e.g. -DTM_MUTATE=1);
    such builds never replace the product library."""
    extra = list(extra or [])
    if verbose:
        extra += ["-Xptxas", "-v"]
    if out is not None:
        return _build_to(out, extra)
    if not force and not _stale(extra):
        return LIB
    import tempfile
    os.makedirs(OUT_DIR, exist_ok=True)
    with tempfile.TemporaryDirectory(prefix="tm_build_", dir=OUT_DIR) as obj_dir:
        with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
            done = list(ex.map(lambda s: _compile(s, extra, obj_dir), SOURCES))
        objs = [o for o, _ in done]
        tmp = LIB + f".tmp{os.getpid()}"
        link = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", tmp, "-ldl"]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        ver = subprocess.run([NVCC, "--version"], capture_output=True, text=True).stdout.strip().splitlines()[-1:]
        stamp = {"source_sha256": _source_hash(extra), "nvcc": ver, "compile": [c for _, c in done], "link": link}
        os.replace(tmp, LIB)
        with open(STAMP, "w") as f:
            json.dump(stamp, f, indent=1)
    return LIB


def _build_to(out: str, extra: list[str]) -> str:
    import tempfile
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    with tempfile.TemporaryDirectory(prefix="tm_build_") as obj_dir:
        with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
            objs = [o for o, _ in ex.map(lambda s: _compile(s, extra, obj_dir), SOURCES)]
        link = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", out, "-ldl"]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
