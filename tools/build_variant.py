"""Build an alternative libfvdb_b200.so with extra compile-time defines for one source file (profiling).

python tools/build_variant.py NAME SRC.cu -DFOO=1 ...  -> paper_2407_01781_b200/_lib/variants/libfvdb_b200_NAME.so
Run with FVDB_LIB_VARIANT=NAME to load it (paper_2407_01781_b200/_lib.py).  The other objects are the
in-tree build's (python -m paper_2407_01781_b200._build first).
"""
import pathlib
import subprocess
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2407_01781_b200 import _build as B  # noqa: E402

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
objdir = B.LIBDIR / "obj"
vdir = B.LIBDIR / "variants"
vdir.mkdir(exist_ok=True)
src = B.CSRC / src
obj = vdir / f"{src.stem}_{name}.o"
subprocess.run([B.nvcc(), *B.ARCH, *B.NVCC_FLAGS, *defs, "-c", str(src), "-o", str(obj)], check=True)
objs = [str(obj)] + [str(o) for o in sorted(objdir.glob("*.o")) if o.stem != src.stem]
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", str(vdir / f"libfvdb_b200_{name}.so"), *objs], check=True)
print(vdir / f"libfvdb_b200_{name}.so")
