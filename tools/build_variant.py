"""Build a diagnostic variant of liblhaf.so into build/variants/NAME.so (git-ignored; travels to
the GPU box with the gpurun snapshot) for A/B timing through LHAF_LIB_PATH.
    python tools/build_variant.py NAME [--rev GITREV] [-DFLAG=V ...]
--rev takes csrc/ and include/ from a git revision (e.g. HEAD) instead of the working tree."""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
name = sys.argv[1]
rev = None
flags = []
for a in sys.argv[2:]:
    if a.startswith("--rev="):
        rev = a.split("=", 1)[1]
    else:
        flags.append(a)
tmp = tempfile.mkdtemp()
src = os.path.join(tmp, "pkg", "csrc")
inc = os.path.join(tmp, "include")
if rev:
    os.makedirs(src); os.makedirs(inc)
    for d, out in (("paper_2108_01622_b200/csrc", src), ("include", inc)):
        files = subprocess.check_output(["git", "-C", ROOT, "ls-tree", "--name-only", f"{rev}:{d}"], text=True).split()
        for f in files:
            with open(os.path.join(out, f), "wb") as fh:
                fh.write(subprocess.check_output(["git", "-C", ROOT, "show", f"{rev}:{d}/{f}"]))
else:
    shutil.copytree(os.path.join(ROOT, "paper_2108_01622_b200", "csrc"), src)
    shutil.copytree(os.path.join(ROOT, "include"), inc)
os.makedirs(os.path.join(ROOT, "build", "variants"), exist_ok=True)
out = os.path.join(ROOT, "build", "variants", name + ".so")
srcs = [os.path.join(src, f) for f in ("lhaf_kernels.cu", "lhaf_v3.cu", "lhaf_v5.cu", "lhaf_tree.cu", "lhaf_host.cpp", "lhaf_gbs.cpp")]
cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
       "-Xcompiler", "-fPIC,-O2", *flags, "-shared", "-o", out, *srcs, "-I", inc, "-ldl"]
subprocess.check_call(cmd)
shutil.rmtree(tmp)
print(out)
