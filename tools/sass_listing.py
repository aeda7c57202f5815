"""Committed SASS evidence for the hot-path kernels: dumps
`cuobjdump -sass` of the default sweep kernels from the built library and a
per-kernel instruction-mix summary (loads / stores by width, spills, FP64 /
FP32 arithmetic, branches).

    python tools/sass_listing.py [out_dir]     (default profiles/)
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1007_1388_b200", "liblbm_b200.so")
# the default launch configurations (sweep.cu / sweep_aa.cu launch wrappers, variant 0)
KERNELS = {
    "sweep_x2_fp64": "_ZN3lbm15sweep_x2_kernelIdLi3ELb0EEEvNS_9SweepArgsIT_EE",
    "sweep_x2_fp32": "_ZN3lbm15sweep_x2_kernelIfLi5ELb0EEEvNS_9SweepArgsIT_EE",
    "sweep_x2_direct_fp32": "_ZN3lbm15sweep_x2_kernelIfLi5ELb1EEEvNS_9SweepArgsIT_EE",
    "sweep_aa_pull_fp64": "_ZN3lbm18sweep_aa_x2_kernelIdLb1ELi3ELb0EEEvNS_9SweepArgsIT_EE",
    "sweep_aa_local_fp64": "_ZN3lbm18sweep_aa_x2_kernelIdLb0ELi3ELb0EEEvNS_9SweepArgsIT_EE",
    "bb_list_fp64_mode0": "_ZN3lbm14bb_list_kernelIdLi0EEEvPT_PKhPKNS_7BbEntryElPKS1_NS_4GeomENS_9BbOffsetsENS_7CheckerE",
}


def functions(sass):
    out = {}
    for part in re.split(r"\n\s*Function : ", sass)[1:]:
        name = part.split("\n")[0].strip()
        out[name] = [l for l in part.split("\n") if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
    return out


def mix(lines):
    c = collections.Counter()
    for l in lines:
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", l)
        if not m:
            continue
        op = m.group(2)
        base = op.split(".")[0]
        if base in ("LDG", "STG", "LDL", "STL", "LDS", "STS"):
            c[op] += 1
        elif base in ("DFMA", "DADD", "DMUL", "FFMA", "FADD", "FMUL", "FFMA2", "FADD2", "FMUL2", "BRA", "EXIT", "SEL", "IMAD", "IADD3", "LEA"):
            c[base] += 1
        c["total"] += 1
    return c


def main():
    out_dir = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles")
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    fns = functions(sass)
    summary = []
    for tag, name in KERNELS.items():
        lines = fns.get(name)
        if lines is None:
            summary.append(f"{tag}: {name} not found")
            continue
        with open(os.path.join(out_dir, f"r02_sass_{tag}.txt"), "w") as fh:
            fh.write(f"// cuobjdump -sass {os.path.relpath(LIB, ROOT)} -- {name}\n")
            fh.write("\n".join(lines) + "\n")
        c = mix(lines)
        summary.append(f"{tag} ({name}): " + ", ".join(f"{k}={v}" for k, v in sorted(c.items())))
    with open(os.path.join(out_dir, "r02_sass_summary.txt"), "w") as fh:
        fh.write("# static instruction mix of the default hot-path kernels (tools/sass_listing.py)\n")
        fh.write("\n".join(summary) + "\n")
    print("\n".join(summary))


if __name__ == "__main__":
    main()
