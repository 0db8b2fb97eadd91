"""Build a variant libtgp.so with extra -D flags into variants/<name>/libtgp.so (experiments only; load
it with TGP_LIB=...).   python profiles/build_variant.py NAME -DFOO=1 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2004_09910_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
b.FLAGS = b.FLAGS + defs
b.OBJ = os.path.join(root, "build", "obj_" + name)
b.OUT = os.path.join(root, "variants", name, "libtgp.so")
os.makedirs(os.path.dirname(b.OUT), exist_ok=True)
b.build()
