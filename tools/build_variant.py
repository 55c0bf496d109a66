"""Build a tuning variant of libatos.so with extra -D flags (experiments only).

usage: python tools/build_variant.py TAG -DFOO=1 ...  ->  paper_2112_00132_b200/variants/libatos_TAG.so
Run it with ATOS_LIB=<that path> (the binding loads it instead of the product
library, which is never overwritten).
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_00132_b200 import build as b  # noqa: E402

tag, flags = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(b.HERE, "variants")
os.makedirs(out_dir, exist_ok=True)
out = os.path.join(out_dir, f"libatos_{tag}.so")
cmd = [b.nvcc(), *b.NVCC_FLAGS, *flags, "-I", os.path.join(b.ROOT, "include"), "-o", out, *b.sources(), "-ldl"]
subprocess.check_call(cmd)
print(out)
