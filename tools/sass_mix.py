"""SASS instruction mix of the hot kernels (2048-bit size class) from the
built library: per kernel the instruction count, the IMAD.WIDE share (one
32×32→64 product per instruction), other integer ops, shuffles, shared and
global loads, local-memory traffic (spills) and the register count.  Static
counts (each instruction once, loops not unrolled further) — a check that
the inner loops are IMAD.WIDE carry chains without spills or IMAD.MOV.

    python tools/sass_mix.py [lib] > profiles/r02_sass_mix.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2504_03909_b200", "lib", "libsfxb_cuda.so")
KERNELS = [
    ("K2 passive party (base-n digits)", r"k_seg_prod_nd<64, 4, 64>"),
    ("K2 key holder (CRT base-p digits)", r"k_seg_prod_p2<32, 1, 64>"),
    ("K2 mod-n^2 CIOS (fallback)", r"k_seg_prod<128, 4, 64>"),
    ("K1 encrypt step 1 (mod p)", r"k_enc_step1<32, 1, 5>"),
    ("K1 encrypt step 2 (x^p mod p^2, digits)", r"k_p2_pow<32, 1, 5, 0>"),
    ("K3 decrypt (c^(p-1) mod p^2, digits)", r"k_p2_pow<32, 1, 5, 1>"),
    ("K2 finalize (key holder)", r"k_hist_finalize_p2<32,"),
]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and cur:
            funcs[cur].append(m.group(1))
    regs = {}
    for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+)\s+STACK:(\d+)\s+SHARED:(\d+)\s+LOCAL:(\d+)", res):
        regs[m.group(1)] = (int(m.group(2)), int(m.group(3)), int(m.group(5)))
    names = list(funcs)
    dem = dict(zip(names, demangle(names)))
    print("| kernel | instance | instr | IMAD.WIDE | IMAD (other) | IADD3/IADD | SHFL | LDS | LDG | LDL/STL | regs | stack/local B |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for label, pat in KERNELS:
        hit = [f for f in names if pat in dem[f]]
        for f in hit[:1]:
            ops = funcs[f]
            c = collections.Counter()
            for o in ops:
                if o.startswith("IMAD.WIDE"):
                    c["wide"] += 1
                elif o.startswith("IMAD"):
                    c["imad"] += 1
                elif o.startswith("IADD"):
                    c["iadd"] += 1
                elif o.startswith("SHFL"):
                    c["shfl"] += 1
                elif o.startswith("LDS"):
                    c["lds"] += 1
                elif o.startswith("LDG"):
                    c["ldg"] += 1
                elif o.startswith("LDL") or o.startswith("STL"):
                    c["local"] += 1
            r = regs.get(f, ("?", "?", "?"))
            inst = dem[f].split("(")[0].replace("void sfxb::dev::", "")
            print(f"| {label} | `{inst}` | {len(ops)} | {c['wide']} ({100 * c['wide'] / max(1, len(ops)):.0f}%) | "
                  f"{c['imad']} | {c['iadd']} | {c['shfl']} | {c['lds']} | {c['ldg']} | {c['local']} | {r[0]} | "
                  f"{r[1]}/{r[2]} |")


if __name__ == "__main__":
    main()
