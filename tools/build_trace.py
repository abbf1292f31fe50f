"""Build ab/trace/libevoformer_sm100.so: the library with a trace define on
one source (phase timestamps for tools/f2_trace.py / tools/gemm_trace.py).

    python tools/build_trace.py [attention_tc_fwd2|gemm_tc|attention_tc_bwd]
"""
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_05477_b200 import build as B  # noqa: E402

DEFINES = {"attention_tc_fwd2": "-DEVO_F2_TRACE", "gemm_tc": "-DEVO_GEMM_TRACE",
           "attention_tc_bwd": "-DEVO_BWD_TRACE"}
which = sys.argv[1] if len(sys.argv) > 1 else "attention_tc_fwd2"
B.build(verbose=False)
os.makedirs("ab/trace", exist_ok=True)
objs = []
for src in sorted(glob.glob(os.path.join(B.CSRC, "*.cu"))):
    o = os.path.join(B.BUILD, os.path.basename(src) + ".o")
    if os.path.basename(src) == which + ".cu":
        o = f"ab/trace/{which}.o"
        subprocess.run([B.NVCC, *B.ARCH, *B.CFLAGS, DEFINES[which], "-c", src, "-o", o], check=True)
    objs.append(o)
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", "ab/trace/libevoformer_sm100.so", *objs, "-cudart", "static"],
               check=True)
print("built ab/trace/libevoformer_sm100.so with", DEFINES[which])
