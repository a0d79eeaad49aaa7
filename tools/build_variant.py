"""Build an A/B variant of libcusci.so with extra nvcc flags into tools/variants/NAME.so:
    python tools/build_variant.py NAME -DFOO=1 ...   (then tools/variant_run.sh "CMD")"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_15768_b200 import build as b  # noqa: E402

os.makedirs(os.path.join(ROOT, "tools", "variants"), exist_ok=True)
print(b.build(force=True, out=os.path.join(ROOT, "tools", "variants", sys.argv[1] + ".so"), extra=sys.argv[2:]))
