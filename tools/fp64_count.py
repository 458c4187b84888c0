"""FP64 arithmetic instructions (DFMA/DMUL/DADD, thread-level, executed) per
cell of one stage-kernel launch, from the ncu SASS source page.

usage: python tools/fp64_count.py REPORT.ncu-rep KERNEL_SUBSTRING CELLS"""
import collections
import sys



def blocks(rep, ksub):
    import csv
    import subprocess

    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    res, cur = [], None
    for r in csv.reader(out.splitlines()):
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            res.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None:
            cur["rows"].append(r)
    return [b for b in res if ksub in b["name"]]


def main():
    rep, ksub, cells = sys.argv[1], sys.argv[2], float(sys.argv[3])
    for i, b in enumerate(blocks(rep, ksub)):
        print(f"launch {i}: {b['name'][:60]}")
        count(b, cells)


def count(b, cells):
    ci = {h: i for i, h in enumerate(b["hdr"])}
    cnt = collections.Counter()
    for r in b["rows"]:
        if len(r) < len(b["hdr"]):
            continue
        parts = r[ci["Source"]].split()
        if not parts:
            continue
        op = (parts[1] if parts[0].startswith("@") else parts[0]).split(".")[0]
        try:
            n = float(r[ci["Thread Instructions Executed"]] or 0)
        except ValueError:
            continue
        cnt[op] += n
    fp64 = sum(cnt[o] for o in ("DFMA", "DMUL", "DADD"))
    tot = sum(cnt.values())
    print(f"fp64 (DFMA+DMUL+DADD) per cell: {fp64 / cells:.1f}; all thread instructions per cell: {tot / cells:.1f}")
    for o, n in cnt.most_common(20):
        print(f"  {o:10s} {n / cells:8.1f}")


if __name__ == "__main__":
    main()
