"""Build a tuning variant of libnsp.so with extra -D defines into tools/variants/<name>/libnsp.so
(diagnostics; the product library is paper_2101_12164_b200/libnsp.so).  Select it at run time with
NSP_LIB=tools/variants/<name>/libnsp.so.
    python tools/build_variant.py NAME -DNSP_PANEL_NW=8 ..."""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2101_12164_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "tools", "variants", name)
os.makedirs(out, exist_ok=True)


def comp(src):
    obj = os.path.join(out, os.path.splitext(src)[0] + ".o")
    lang = [] if src.endswith(".cu") else ["-x", "cu"]
    cmd = [B.NVCC, *B.ARCH, *B.FLAGS, *defs, *lang, "-c", os.path.join(B.CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    return obj


with cf.ThreadPoolExecutor(len(B.SOURCES)) as ex:
    objs = list(ex.map(comp, B.SOURCES))
r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", os.path.join(out, "libnsp.so"), *objs,
                    "-Xcompiler", "-fopenmp", "-lgomp", "-ldl"], capture_output=True, text=True)
if r.returncode:
    raise RuntimeError(r.stderr)
print("built", os.path.join(out, "libnsp.so"))
