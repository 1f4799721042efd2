"""Build an A/B variant of libfsp.so with extra nvcc defines (diagnostics):
python tools/build_variant.py NAME -DFOO=1 ...  ->  _build/variants/libfsp_NAME.so,
loaded by the binding when FSP_LIB_VARIANT=NAME."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1208_3933_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(b.BUILD, "variants")
os.makedirs(out, exist_ok=True)
objs = []
for src in b.sources():
    obj = os.path.join(out, f"{name}_{os.path.basename(src)}.o")
    subprocess.check_call([b.NVCC, *b.ARCH, *b.FLAGS, *defs, "-I", b.INCLUDE, "-I", b.CSRC, "-c", src, "-o", obj],
                          stderr=subprocess.DEVNULL)
    objs.append(obj)
subprocess.check_call([b.NVCC, *b.ARCH, "-shared", "-o", os.path.join(out, f"libfsp_{name}.so"), *objs,
                       "-lcudart_static", "-lrt", "-ldl", "-lpthread"])
print(os.path.join(out, f"libfsp_{name}.so"))
