"""Build a variant of libsgs.so with extra nvcc defines into its own build dir
(A/B experiments through SGS_LIB_PATH, tools/ab.sh):
    python tools/build_variant.py abtest/libsgs_pf4.so -DSGS_ATTN_PF=4"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_15930_b200 import build as B  # noqa: E402

out, defs = os.path.abspath(sys.argv[1]), sys.argv[2:]
tag = os.path.splitext(os.path.basename(out))[0]
B.COMMON = B.COMMON + defs
B.BUILD = os.path.join(ROOT, "build", "variant_" + tag)
B.LIB = out
os.makedirs(os.path.dirname(out), exist_ok=True)
B.build(force=True, verbose=True)
