"""Build a tuning variant of libpuzzlemoe.so: one csrc file recompiled with extra -D flags,
linked with the other objects of the in-tree build.

    python scripts/build_variant.py NAME FILE.cu[,FILE2.cu] -DKNOB=VALUE ...
    -> build/variants/NAME/libpuzzlemoe.so   (load it with PUZZLE_LIB=<that path>)"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_04805_b200 import build as B  # noqa: E402

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
out = os.path.join(B.ROOT, "build", "variants", name)
os.makedirs(out, exist_ok=True)
rebuilt = {}
for one in src.split(","):
    obj = os.path.join(out, one[:-3] + ".o")
    subprocess.check_call([B.NVCC, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, one), "-o", obj],
                          stderr=subprocess.DEVNULL)
    rebuilt[os.path.basename(obj)] = obj
objs = [rebuilt.get(os.path.basename(o), o)
        for o in (os.path.join(B.BUILD, os.path.basename(s)[:-3] + ".o") for s in B._sources())]
subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", os.path.join(out, "libpuzzlemoe.so"), *objs,
                       "-cudart", "static", "-Xlinker", "--no-undefined"])
print(os.path.join(out, "libpuzzlemoe.so"))
