"""Experiment builds (timing only, never the product library): compile every
source once into _exp/obj, then for each variant recompile the named sources
with extra -D flags and link _exp/libtm_<name>.so (load with TM_LIB_PATH).
usage: build_variants.py name:src1,src2:-DFOO=1[:-DBAR=2] ..."""
import concurrent.futures as cf, os, subprocess, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_1804_10694_b200 import _build as B

EXP = os.path.join(B.ROOT, "_exp")
OBJ = os.path.join(EXP, "obj")
os.makedirs(OBJ, exist_ok=True)
with cf.ThreadPoolExecutor(len(B.SOURCES)) as ex:
    base = dict(zip(B.SOURCES, [o for o, _ in ex.map(lambda s: B._compile(s, [], OBJ), B.SOURCES)]))


def variant(spec):
    name, srcs, *flags = spec.split(":")
    d = os.path.join(EXP, "obj_" + name)
    os.makedirs(d, exist_ok=True)
    objs = dict(base)
    for s in srcs.split(","):
        objs[s] = B._compile(s, flags, d)[0]
    out = os.path.join(EXP, f"libtm_{name}.so")
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-Xcompiler", "-fPIC", *objs.values(), "-o", out, "-ldl"], check=True)
    return out


with cf.ThreadPoolExecutor(4) as ex:
    for o in ex.map(variant, sys.argv[1:]):
        print(o)
