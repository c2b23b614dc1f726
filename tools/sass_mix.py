"""Static SASS instruction mix per kernel of an object file (FP vs integer/ALU vs smem).

Usage:  python tools/sass_mix.py OBJ.o [name-regex]
"""
import re
import subprocess
import sys
from collections import Counter

ALU = {"LEA", "LOP3", "IADD3", "SHF", "ISETP", "FSEL", "FSETP", "SEL", "IMNMX", "FMNMX", "PLOP3", "VIADD", "IABS"}
FP = {"FFMA", "FADD", "FMUL", "FFMA2", "FADD2", "FMUL2"}


def main():
    obj = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    fn, mix = None, {}
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            mix[fn] = Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if fn and m:
            mix[fn][m.group(1)] += 1
    for fn, c in mix.items():
        name = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
        if pat and not pat.search(name):
            continue
        alu = sum(v for k, v in c.items() if k in ALU)
        fp = sum(v for k, v in c.items() if k in FP)
        sm = c["LDS"] + c["STS"]
        print(f"{sum(c.values()):6d} total {fp:5d} fp {alu:5d} alu {c['IMAD']:4d} imad {sm:4d} lds/sts  "
              f"{name.replace('mgb::(anonymous namespace)::', '')[:70]}")


if __name__ == "__main__":
    main()
