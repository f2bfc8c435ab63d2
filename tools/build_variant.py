"""Build the engine with extra nvcc flags into tools/altlibs/<name>.so (A/B and instrumented
builds; run with ITERCUR_LIB_OVERRIDE=tools/altlibs/<name>.so). Example:
    python tools/build_variant.py instr -DITERCUR_LUPP_INSTRUMENT"""
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_21963_b200 import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(ROOT, "tools", "altlibs", "obj_" + name)
os.makedirs(out_dir, exist_ok=True)


def comp(src):
    obj = os.path.join(out_dir, os.path.basename(src)[:-3] + ".o")
    cmd = [B.NVCC, *B.ARCH, *extra, *B.FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    return obj


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(comp, sorted(glob.glob(os.path.join(B.CSRC, "*.cu")))))
lib = os.path.join(ROOT, "tools", "altlibs", name + ".so")
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs], check=True)
print(lib)
