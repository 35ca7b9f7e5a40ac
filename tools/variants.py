"""Build libhegpu.so variants that differ only in eval.cu compile-time
macros (e.g. HEGPU_HS_BT, HEGPU_HS_MINB), for A/B timing on the GPU box:
  python tools/variants.py NAME:-DX=1,-DY=2 ...   -> tools/bin/libhegpu_NAME.so
then  HEGPU_LIB=tools/bin/libhegpu_NAME.so python bench.py ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_08321_b200 import build as B  # noqa: E402

B.build()
objs = [os.path.join(B.OBJ, f) for f in sorted(os.listdir(B.OBJ)) if f.endswith(".o")]
os.makedirs(os.path.join(ROOT, "tools", "bin"), exist_ok=True)
for spec in sys.argv[1:]:
    name, _, flags = spec.partition(":")
    flags = [f for f in flags.split(",") if f]
    srcs = os.environ.get("VARIANT_SRC", "eval.cu").split(",")
    vobjs = []
    for src in srcs:
        obj = f"/tmp/var/{src}_{name}.o"
        cmd = [B.NVCC, *B.ARCH, *B.COMMON, *flags, "-c", os.path.join(B.CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd = [B.NVCC, *B.COMMON, *flags, "-x", "c++", "-c", os.path.join(B.CSRC, src), "-o", obj]
        subprocess.run(cmd, check=True)
        vobjs.append(obj)
    lib = os.path.join(ROOT, "tools", "bin", f"libhegpu_{name}.so")
    link = [o for o in objs if not any(o.endswith(src + ".o") for src in srcs)] + vobjs
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *link, "-Xcompiler", "-fopenmp", "-lgomp", "-lcudart"],
                   check=True)
    print(lib)
