"""Static SASS opcode histogram of a kernel's main loop (design experiments).

    python tools/sass_loop.py CUBIN KERNEL_SUBSTRING

The main loop is taken as the span of the backward branch that covers the most
instructions.  Also prints the registers / spills of the kernel.
"""
import collections
import re
import subprocess
import sys


def main():
    cubin, sub = sys.argv[1], sys.argv[2]
    out = subprocess.check_output(["cuobjdump", "-sass", cubin], text=True)
    funcs = re.split(r"\n\s+Function : ", out)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if sub not in name:
            continue
        ins = []
        for line in f.split("\n"):
            m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2)))
        best = None
        for a, t in ins:
            m = re.search(r"BRA(?:\.\w+)*\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)", t)
            if m and int(m.group(1), 16) < a:
                span = (int(m.group(1), 16), a)
                if best is None or span[1] - span[0] > best[1] - best[0]:
                    best = span
        c = collections.Counter()
        for a, t in ins:
            if best and best[0] <= a <= best[1]:
                op = t.split()[1] if t.startswith("@") else t.split()[0]
                c[op.split(".")[0]] += 1
        print(name)
        print(f"  total {len(ins)}  loop {sum(c.values())}  [{best[0]:#x}, {best[1]:#x}]" if best else "  no loop")
        fp64 = sum(c[k] for k in ("DFMA", "DMUL", "DADD"))
        print(f"  loop fp64 {fp64}  fsel {c['FSEL']}  mufu {c['MUFU']}  lds {c['LDS']}  sts {c['STS']}  bar {c['BAR']}")
        print("  " + "  ".join(f"{k} {v}" for k, v in c.most_common(30)))


if __name__ == "__main__":
    main()
