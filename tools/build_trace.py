"""Build ab/trace/libevoformer_sm100.so: the library with -DEVO_F2_TRACE on
attention_tc_fwd2.cu (phase timestamps for tools/f2_trace.py)."""
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import build as B  # noqa: E402

B.build(verbose=False)
os.makedirs("ab/trace", exist_ok=True)
objs = []
for src in sorted(glob.glob(os.path.join(B.CSRC, "*.cu"))):
    o = os.path.join(B.BUILD, os.path.basename(src) + ".o")
    if "attention_tc_fwd2" in src:
        o = "ab/trace/f2.o"
        subprocess.run([B.NVCC, *B.ARCH, *B.CFLAGS, "-DEVO_F2_TRACE", "-c", src, "-o", o], check=True)
    objs.append(o)
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", "ab/trace/libevoformer_sm100.so", *objs, "-cudart", "static"],
               check=True)
print("built ab/trace/libevoformer_sm100.so")
