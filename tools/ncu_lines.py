"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

usage: python tools/ncu_lines.py REPORT.ncu-rep CUBIN KERNEL_SUBSTRING [TOP]
(extract the cubin with `cuobjdump -xelf all libspark.so` in a scratch dir; the
report must come from the same build)."""
import collections
import csv
import re
import subprocess
import sys


def sass_rows(rep, ksub):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks, cur = [], None
    for r in csv.reader(out.splitlines()):
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None:
            cur["rows"].append(r)
    for b in blocks:
        if ksub in b["name"]:
            return b
    raise SystemExit(f"kernel {ksub} not in report: {[b['name'][:80] for b in blocks]}")


def line_map(cubin, mangled_sub):
    names = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True).stdout
    funcs = re.findall(r"Function : (\S+)", names)
    cands = [f for f in funcs if all(s in f for s in mangled_sub)]
    if not cands:
        raise SystemExit(f"no function matching {mangled_sub}")
    fn = cands[0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    m, cur, inside = {}, None, False
    for ln in dis.splitlines():
        if ".section" in ln and ".text." in ln:
            inside = fn in ln
            continue
        if not inside:
            continue
        mm = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if mm:
            cur = (mm.group(1).split("/")[-1], int(mm.group(2)))
            continue
        mi = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if mi and cur:
            m[int(mi.group(1), 16)] = cur
    return fn, m


def main():
    rep, cubin, ksub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    b = sass_rows(rep, ksub)
    hdr = b["hdr"]
    ci = {h: i for i, h in enumerate(hdr)}
    # template args "<(int)3, (int)1, (int)1, (int)16, (int)16>" -> mangled "ILi3ELi1ELi1ELi16ELi16E"
    targs = re.findall(r"\(int\)(\d+)", b["name"])
    kname = re.search(r"::(\w+)<", b["name"]).group(1)  # e.g. stage_kernel, amr_leaf_kernel
    fn, lm = line_map(cubin, [kname, "I" + "".join(f"Li{a}E" for a in targs)])
    samples = collections.Counter()
    stall = collections.defaultdict(collections.Counter)
    execd = collections.Counter()
    total = 0.0
    base = None
    for r in b["rows"]:
        try:
            a = int(r[ci["Address"]], 16)
            base = a if base is None else min(base, a)
        except (ValueError, IndexError):
            pass
    for r in b["rows"]:
        if len(r) < len(hdr):
            continue
        try:
            addr = int(r[ci["Address"]], 16) - base
            s = float(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        key = lm.get(addr, ("?", 0))
        samples[key] += s
        total += s
        execd[key] += float(r[ci["Instructions Executed"]] or 0)
        for h in hdr:
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    v = float(r[ci[h]] or 0)
                except ValueError:
                    v = 0
                if v:
                    stall[key][h[6:]] += v
    srcs = {}
    for (f, ln), s in samples.most_common(top):
        if f not in srcs:
            path = {"spark_stage.cu": "paper_2401_03378_b200/csrc/spark_stage.cu",
                    "spark_device.cuh": "paper_2401_03378_b200/csrc/spark_device.cuh"}.get(f)
            srcs[f] = open(path).read().splitlines() if path else []
        text = srcs[f][ln - 1].strip()[:70] if srcs[f] and 0 < ln <= len(srcs[f]) else ""
        st = ", ".join(f"{k}:{v / s * 100:.0f}%" for k, v in stall[(f, ln)].most_common(3))
        print(f"{s / total * 100:5.1f}%  {f}:{ln:<4d} exec {execd[(f, ln)] / 1e6:6.1f}M  [{st}]  {text}")


if __name__ == "__main__":
    main()
