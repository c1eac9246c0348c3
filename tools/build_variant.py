"""Build an experiment variant of libsw_plan.so with extra -D defines (same ABI), loaded by
setting SW_LIB_VARIANT=NAME.  usage: python tools/build_variant.py NAME DEF=VAL ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_05800_b200 import build  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
d = os.path.join(build.PKG, "variants")
os.makedirs(d, exist_ok=True)
print(build.build(force=True, out=os.path.join(d, "libsw_plan_%s.so" % name), defines=defs))
