"""SASS instruction histogram of the hot kernels (static counts from cuobjdump of
the in-tree objects) -> profiles/sass_hist_<round>.md.  Shows the fp64 work
(DFMA / DMUL / DADD), the FP64 tensor-core DMMA, spills (STL / LDL), shared
memory traffic and the uniform-datapath constant materialisation (UMOV / LDCU).

    python tools/sass_hist.py [round]
"""
import re
import subprocess
import sys
from collections import Counter

ROUND = sys.argv[1] if len(sys.argv) > 1 else "r02"
OBJ = "paper_2403_01521_b200/_lib/obj"
KERNELS = [
    ("fourier.o", "fourier_sweep_kernelILi8ELb0E", "fourier_sweep_kernel<8>"),
    ("fourier.o", "fourier_aggregate_mma_kernelILi8E", "fourier_aggregate_mma_kernel<8>"),
    ("fourier.o", "fourier_carry_compose_kernel", "fourier_carry_compose_kernel"),
    ("zero.o", "zero_sweep_kernelILi8E", "zero_sweep_kernel<8>"),
    ("short.o", "pair_list_kernelILi2ELi1E", "pair_list_kernel<2,1>"),
    ("short.o", "nbr_build_kernelILi3E", "nbr_build_kernel<3>"),
    ("short_tile.o", "short_tile_kernelILb1E", "short_tile_kernel<true>"),
    ("sort.o", "radix_onesweep_kernelImLi16E", "radix_onesweep_kernel<u64,16>"),
]
CLASSES = ["DFMA", "DMUL", "DADD", "DMMA", "FFMA2", "FADD2", "FFMA", "FADD", "FMUL", "MUFU",
           "LDS", "STS", "LDG", "STG", "LDL", "STL", "SHFL", "UMOV", "LDCU", "IMAD", "LOP3",
           "FSEL", "BRA"]


def sass(obj):
    return subprocess.run(["cuobjdump", "-sass", f"{OBJ}/{obj}"], capture_output=True,
                          text=True, check=True).stdout


def functions(text):
    cur, out = None, {}
    for line in text.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            out[cur] = []
        elif cur and re.search(r"/\*[0-9a-f]{4}\*/", line):
            out[cur].append(line)
    return out


def main():
    cache = {}
    rows = []
    for obj, key, label in KERNELS:
        if obj not in cache:
            cache[obj] = functions(sass(obj))
        name = next((f for f in cache[obj] if key in f), None)
        if name is None:
            continue
        c = Counter()
        for line in cache[obj][name]:
            m = re.search(r"\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
            if m:
                c[m.group(2)] += 1
        rows.append((label, sum(c.values()), c))
    out = [f"# SASS instruction histogram, round {ROUND}", "",
           "Static counts per kernel (whole function, all paths) from `cuobjdump -sass` of the "
           "sm_100a objects (`tools/sass_hist.py`).  DMMA = FP64 tensor core (`mma.sync` "
           "m8n8k4); FFMA2/FADD2 = paired fp32; LDL/STL = spills.", "",
           "| kernel | total | " + " | ".join(CLASSES) + " |",
           "|---|---:|" + "---:|" * len(CLASSES)]
    for label, tot, c in rows:
        out.append(f"| {label} | {tot} | " + " | ".join(str(c.get(k, 0)) for k in CLASSES) + " |")
    text = "\n".join(out) + "\n"
    with open(f"profiles/sass_hist_{ROUND}.md", "w") as fh:
        fh.write(text)
    print(text)


if __name__ == "__main__":
    main()
