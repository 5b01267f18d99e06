"""Build a library from the current csrc with some files replaced (A/B of kernel rewrites):
python tools/build_mix.py out.so file.cu=/path/to/alt.cu ..."""
import os, shutil, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2009_04061_b200 import build as b
out = os.path.abspath(sys.argv[1])
tmp = tempfile.mkdtemp()
shutil.copytree(os.path.join(ROOT, "paper_2009_04061_b200", "csrc"), os.path.join(tmp, "pkg", "csrc"))
shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
for spec in sys.argv[2:]:
    name, alt = spec.split("=")
    shutil.copy(alt, os.path.join(tmp, "pkg", "csrc", name))
objs = []
for src in b.SOURCES:
    o = os.path.join(tmp, src.replace(".cu", ".o"))
    subprocess.check_call(["nvcc", *b.ARCH, *b.FLAGS, "-c", os.path.join(tmp, "pkg", "csrc", src), "-o", o],
                          stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    objs.append(o)
subprocess.check_call(["nvcc", *b.ARCH, "-shared", "-o", out, *objs])
shutil.rmtree(tmp)
print(out)
