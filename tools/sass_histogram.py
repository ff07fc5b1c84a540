"""SASS instruction histogram of the shipped library (cuobjdump -sass; runs without a GPU). Proves the
Blackwell-native instruction mix per kernel: UTCHMMA (tcgen05.mma), LDTM/STTM (TMEM), UBLKCP (bulk-async
copy engine), SYNCS (mbarriers), MUFU, FFMA2. python tools/sass_histogram.py [lib] > profiles/r02/sass_histogram.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEY = ["UTCHMMA", "UTCHMMA.2CTA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "SYNCS", "MUFU.TANH", "MUFU.EX2", "MUFU.LG2",
       "MUFU.SIN", "MUFU.COS", "MUFU.RSQ", "FFMA2", "FFMA", "FADD", "F2FP", "LDS", "STS", "LDG", "STG", "LDL", "STL",
       "ELECT", "USETMAXREG", "BAR", "SHFL"]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2603_07199_b200", "libmppi_b200.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and cur:
            op = m.group(2)
            kernels[cur][op] += 1
    dem = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True, text=True).stdout.splitlines()
    print(f"# SASS histogram of {os.path.relpath(lib, ROOT)} ({len(kernels)} kernels); static instruction counts")
    tot = collections.Counter()
    for (k, c), name in zip(kernels.items(), dem):
        for op, n in c.items():
            tot[op] += n
    print("## whole library:", ", ".join(f"{k} {sum(n for op, n in tot.items() if op == k or op.startswith(k + '.'))}"
                                          for k in KEY))
    for (k, c), name in zip(kernels.items(), dem):
        if not re.search(r"k_mlp_tc<256, 3, 2, 0>|k_mlp_h128<2, 1, 0>|k_mlp_h128<2, 1, 4>|k_rollout<true>|k_softmin<512>|k_mlp_simt<64>", name):
            continue
        print(f"\n## {name[:110]}  ({sum(c.values())} instructions)")
        row = []
        for key in KEY:
            n = sum(v for op, v in c.items() if op == key or op.startswith(key + "."))
            if key == "FFMA":
                n = c["FFMA"]
            if key == "UTCHMMA":
                n = c["UTCHMMA"]
            if n:
                row.append(f"{key} {n}")
        print("   key:", ", ".join(row))
        print("   top:", ", ".join(f"{op} {n}" for op, n in c.most_common(14)))


if __name__ == "__main__":
    main()
