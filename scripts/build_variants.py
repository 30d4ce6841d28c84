"""Build profiling variants of libbt_b200.so: bt_stencil.cu recompiled with extra -D flags, linked against the
product's other objects. Usage: python scripts/build_variants.py s4=-DBT_STAGES=4 ft64="-DBT_FT=64 -DBT_ST16=1" ...
Outputs paper_2308_01792_b200/variants/libbt_<name>.so (git-ignored; they travel to the GPU box). Run with
BT_LIB_PATH=<that file>."""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2308_01792_b200"))
import build as B  # noqa: E402


def one(spec):
    name, flags = spec.split("=", 1)
    src = os.environ.get("BT_VARIANT_SRC", "bt_stencil.cu")
    out_dir = os.path.join(B.PKG, "variants")
    os.makedirs(out_dir, exist_ok=True)
    o = os.path.join(out_dir, f"{src}.{name}.o")
    subprocess.run([B.NVCC, *B.ARCH, *B.CU_FLAGS, *flags.split(), "-c", os.path.join(B.CSRC, src), "-o", o],
                   check=True, capture_output=True)
    objs = [os.path.join(B.OBJ, s + ".o") for s in B.CU_SOURCES + B.CXX_SOURCES if s != src] + [o]
    so = os.path.join(out_dir, f"libbt_{name}.so")
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", so, *objs, "-lcudart_static", "-lrt", "-lpthread", "-ldl"],
                   check=True)
    return so


if __name__ == "__main__":
    B.build()
    with cf.ThreadPoolExecutor(8) as ex:
        for so in ex.map(one, sys.argv[1:]):
            print(so)
