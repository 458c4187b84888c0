"""Write profiles/ncu_summary.json (the numbers bench.py reads) from the two
`ncu --set full` captures of tools/profile.sh (PLM: stages 1-2 of a step;
WENO5/RK3: stages 2-3, stage 1 taken from the PLM capture — same one-read /
one-write pattern).

    python tools/make_ncu_summary.py PLM.ncu-rep WENO.ncu-rep SOURCE_NOTE
"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from fp64_count import blocks  # noqa: E402
from ncu_summary import summarise  # noqa: E402

CELLS = 256 ** 3
NV = 5


def per_zone(b):
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
            cnt[op] += float(r[ci["Thread Instructions Executed"]] or 0)
        except ValueError:
            pass
    return sum(cnt[o] for o in ("DFMA", "DMUL", "DADD")) / CELLS, sum(cnt.values()) / CELLS


def one(rep, stages, S):
    s = [d for d in summarise(rep) if "stage_kernel" in d["kernel"]]
    bl = blocks(rep, "stage_kernel")[::2]  # the source page lists each launch twice
    fp = [round(per_zone(b)[0], 1) for b in bl]
    it = [round(per_zone(b)[1], 1) for b in bl]
    dram = [d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in s]
    ms = [d["gpu__time_duration.sum"] * 1e3 for d in s]
    alg = CELLS * NV * 8 * (2 + 3 * (S - 1)) / S  # stage 1 reads 1, writes 1; later stages read 2
    return {"captured": dram, "stages_captured": stages, "stage_ms": ms, "algorithmic_bytes_per_launch": alg,
            "fp64_inst_per_zone_by_stage": fp, "inst_per_zone_by_stage": it}


def main():
    plm, weno, note = sys.argv[1], sys.argv[2], sys.argv[3]
    p = one(plm, [1, 2], 2)
    w = one(weno, [2, 3], 3)
    p["dram_bytes_per_launch"] = sum(p["captured"]) / len(p["captured"])
    # RK3 step: stage 1 (as the PLM stage-1 capture) + the two captured stages
    w["dram_bytes_per_launch"] = (p["captured"][0] + sum(w["captured"])) / 3
    for d in (p, w):
        fp, it = d["fp64_inst_per_zone_by_stage"], d["inst_per_zone_by_stage"]
        d["fp64_inst_per_zone"] = round(sum(fp) / len(fp), 1)
        d["inst_per_zone"] = round(sum(it) / len(it), 1)
    w["note"] = "stage-1 traffic taken from the PLM stage-1 capture (identical read/write pattern)"
    out = {"_source": note, "c4_sedov3d_plm": p, "c4_sedov3d_weno": w,
           "_fp64_note": "fp64_inst_per_zone = executed DFMA+DMUL+DADD thread instructions per cell per stage "
                         "(the last stage carries the fused CFL epilogue), averaged over the captured stages",
           "_inst_note": "inst_per_zone = all executed thread-level SASS instructions per cell per stage"}
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_summary.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
