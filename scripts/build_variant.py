"""Build a variant of librtgs.so with extra -D flags into a given path (A/B experiments, stats builds).
python scripts/build_variant.py OUT.so [-DNAME[=V] ...]"""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_19706_b200 import build as B  # noqa: E402

out, defs = sys.argv[1], sys.argv[2:]
B.FLAGS = B.FLAGS + defs
B.BUILD = tempfile.mkdtemp(prefix="rtgs_var_")
B.LIB = os.path.abspath(out)
print(B.build(force=True))
