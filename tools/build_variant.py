"""Build a kernel variant of libdgtau.so for A/B timing: dgtau.cu recompiled
with extra -D flags, linked with the in-tree residual-instance objects, into
paper_2210_03523_b200/variants/libdgtau_<name>.so (git-ignored; load it with
DGTAU_SO=... ).  Usage: python tools/build_variant.py NAME [-DFOO=1 ...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_03523_b200 as dg  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
dg.build()
objdir = os.path.join(dg._HERE, "build")
vdir = os.path.join(dg._HERE, "variants")
os.makedirs(vdir, exist_ok=True)
cflags = [f for f in dg.NVCC_FLAGS if f != "-shared"]
obj = os.path.join(objdir, f"dgtau_{name}.o")
subprocess.check_call(["nvcc", *cflags, *defs, "-c", os.path.join(dg._CSRC, "dgtau.cu"), "-o", obj])
objs = [obj, os.path.join(objdir, "basis.cpp.o")] + [os.path.join(objdir, f"res_inst_{k}.cu.o") for k in range(1, 9)]
so = os.path.join(vdir, f"libdgtau_{name}.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", so, *objs])
print(so)
