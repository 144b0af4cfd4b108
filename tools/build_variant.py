"""Build an in-tree measurement variant libvks_<name>.so with extra nvcc flags (e.g. -DVKS_SORT_ITEMS=32),
loaded by the binding when VKS_LIB_VARIANT=<name> is set.  usage: python tools/build_variant.py name flags..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2605_00219_b200"))
import _build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
bdir = os.path.join(ROOT, "build", f"vks_{name}")
os.makedirs(bdir, exist_ok=True)
objs = []
for src in B.SOURCES:
    obj = os.path.join(bdir, src.replace(".cu", ".o"))
    cmd = [B.nvcc(), *B.ARCH, *B.COMMON, *flags, "-c", os.path.join(B.CSRC, src), "-o", obj]
    if src in B.PINNED:
        cmd.insert(1, "-fmad=false")
    subprocess.check_call(cmd)
    objs.append(obj)
lib = os.path.join(B.HERE, f"libvks_{name}.so")
subprocess.check_call([B.nvcc(), *B.ARCH, "-shared", "-o", lib, *objs, "-cudart", "static"])
print(lib)
