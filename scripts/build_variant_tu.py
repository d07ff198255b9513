"""Fast A/B variants: recompile only the named translation units with extra -D defines and link them with
cached objects of the default build (scripts/variants.sh runs the resulting .so files).

    python scripts/build_variant_tu.py NAME TU[,TU...] [DEFINE ...]   -> paper_2604_17172_b200/variants/NAME.so

The default objects are cached under paper_2604_17172_b200/build/default/ (rebuilt when a source is newer).
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_17172_b200 import _build  # noqa: E402

name, tus, defines = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
cache = os.path.join(_build.HERE, "build", "default")
vdir = os.path.join(_build.HERE, "build", name)
out_dir = os.path.join(_build.HERE, "variants")
for d in (cache, vdir, out_dir):
    os.makedirs(d, exist_ok=True)
newest_dep = max(os.path.getmtime(p) for p in _build.sources() + [os.path.join(_build.CSRC, f) for f in
                                                                  os.listdir(_build.CSRC)])
procs, objs = [], []
for src in _build.sources():
    base = os.path.basename(src)
    if base in tus:
        obj = os.path.join(vdir, base + ".o")
        cmd = [_build.NVCC, *_build.FLAGS, *[f"-D{d}" for d in defines], "-c", "-o", obj, src]
        dflt = os.path.join(cache, base + ".o")  # keep the default cache complete (a later default link)
        if not (os.path.exists(dflt) and os.path.getmtime(dflt) > newest_dep):
            procs.append((subprocess.Popen([_build.NVCC, *_build.FLAGS, "-c", "-o", dflt, src]), None))
    else:
        obj = os.path.join(cache, base + ".o")
        if os.path.exists(obj) and os.path.getmtime(obj) > newest_dep:
            objs.append(obj)
            continue
        cmd = [_build.NVCC, *_build.FLAGS, "-c", "-o", obj, src]
    objs.append(obj)
    procs.append((subprocess.Popen(cmd), cmd))
for p, cmd in procs:
    if p.wait() != 0 and cmd is not None:
        raise subprocess.CalledProcessError(p.returncode, cmd)
lib = os.path.join(out_dir, name + ".so")
subprocess.check_call([_build.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs])
print(lib)
