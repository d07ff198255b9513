"""Build a libuzip variant with extra -D defines for an A/B on the GPU (scripts/variants.sh runs them).

    python scripts/build_variant.py NAME [DEFINE ...]     -> paper_2604_17172_b200/variants/NAME.so
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_17172_b200 import _build  # noqa: E402

name, defines = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(ROOT, "paper_2604_17172_b200", "variants")
os.makedirs(out_dir, exist_ok=True)
print(_build.build(force=True, out=os.path.join(out_dir, name + ".so"), defines=defines))
