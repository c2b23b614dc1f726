"""Registers and spills per kernel from a ptxas -v log (build/device/*.o.ptxas.txt).
Usage: python tools/ptxas_regs.py LOG [name-regex] [--spills]"""
import re
import subprocess
import sys


def parse(path):
    out, fn = {}, None
    for line in open(path):
        m = re.search(r"Compiling entry function '(\S+)'", line) or re.search(r"Function properties for (\S+)", line)
        if m:
            fn = m.group(1)
            out.setdefault(fn, {})
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and fn:
            out[fn]["spill"] = int(m.group(1)) + int(m.group(2))
        m = re.search(r"Used (\d+) registers", line)
        if m and fn:
            out[fn]["regs"] = int(m.group(1))
    return out


def main():
    d = parse(sys.argv[1])
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
    names = subprocess.run(["c++filt"], input="\n".join(d), capture_output=True, text=True).stdout.splitlines()
    for (fn, v), name in zip(d.items(), names):
        name = name.replace("mgb::(anonymous namespace)::", "")
        if pat and not pat.search(name):
            continue
        if "--spills" in sys.argv and not v.get("spill"):
            continue
        print(f"{v.get('regs', 0):4d} regs {v.get('spill', 0):6d} B spill  {name[:110]}")


if __name__ == "__main__":
    main()
