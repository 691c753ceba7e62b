"""Summarise an ncu --set full report by CUDA source line (instructions, stall samples).

    ncu -i rep.ncu-rep --page source --csv --print-source=cuda,sass > src.csv
    python profiles/ncu_lines.py src.csv [top]
"""

import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur_file = None
    hdr = None
    per_line = defaultdict(lambda: [0.0, 0.0, 0.0, ""])  # inst executed, samples, thread inst, src
    line_key = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None:
            continue
        d = dict(zip(hdr, r))
        # rows are either a source line (Line No set) or a sass row under it
        if r[0].strip():
            line_key = (cur_file, int(r[0]))
            per_line[line_key][3] = r[1][:90]
        try:
            ie = float(d.get("Instructions Executed", 0) or 0)
            smp = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
            te = float(d.get("Thread Instructions Executed", 0) or 0)
        except ValueError:
            continue
        if line_key and not r[0].strip():
            per_line[line_key][0] += ie
            per_line[line_key][1] += smp
            per_line[line_key][2] += te
    tot_i = sum(v[0] for v in per_line.values())
    tot_s = sum(v[1] for v in per_line.values())
    print(f"total inst {tot_i:.3e}  samples {tot_s:.0f}")
    for k, v in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:top]:
        act = v[2] / v[0] if v[0] else 0
        print(f"{k[0]:>14}:{k[1]:<4} inst {100*v[0]/tot_i:5.1f}%  stall {100*v[1]/max(tot_s,1):5.1f}%  "
              f"act {act:4.1f}  {v[3]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
