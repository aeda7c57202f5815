"""Build an experimental variant of the product library for A/B timing on the
GPU box (tools/variant_bench.sh): copies paper_1007_1388_b200/csrc to a scratch
directory, applies textual patches from a variant file, and links
build/variants/<name>.so.  Nothing here is part of the product path.

    python tools/build_variant.py <name> <patch.py>
The patch file defines PATCHES = [(file, old, new), ...].
"""
import os
import runpy
import shutil
import subprocess
import sys
import sysconfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    name, patch = sys.argv[1], sys.argv[2]
    src = os.path.join(ROOT, "paper_1007_1388_b200", "csrc")
    work = os.path.join(ROOT, "build", "variants", name + "_src")
    shutil.rmtree(work, ignore_errors=True)
    shutil.copytree(src, work)
    for f, old, new in runpy.run_path(patch)["PATCHES"]:
        p = os.path.join(work, f)
        s = open(p).read()
        assert s.count(old) == 1, (f, old[:60], s.count(old))
        open(p, "w").write(s.replace(old, new))
    nccl = os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl")
    flags = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-Xcompiler", "-fPIC",
             "-Xcompiler", "-fvisibility=hidden", "-I", os.path.join(ROOT, "include"), "-I", nccl + "/include",
             "--expt-relaxed-constexpr"]
    objs = []
    procs = []
    for f in sorted(os.listdir(work)):
        if f.endswith(".cu") or f.endswith(".cpp"):
            o = os.path.join(work, f + ".o")
            cmd = ["nvcc", *flags] + (["-x", "cu"] if f.endswith(".cpp") else []) + ["-c", os.path.join(work, f), "-o", o]
            procs.append(subprocess.Popen(cmd))
            objs.append(o)
    for p in procs:
        assert p.wait() == 0
    out = os.path.join(ROOT, "build", "variants", name + ".so")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out, *objs, "-shared",
                    "-L" + nccl + "/lib", "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nccl + "/lib", "-lcuda"],
                   check=True)
    print(out)


if __name__ == "__main__":
    main()
