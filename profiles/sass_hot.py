"""Per-SASS-instruction execution counts of an ncu --set full report, normalised per
32 walk-steps (one warp-step), hottest-address order preserved.

    ncu -i rep.ncu-rep --page source --csv --print-source sass > sass.csv
    python profiles/sass_hot.py sass.csv <walk_steps_per_launch> > profiles/<tag>_sass.txt
"""

import csv
import sys


def main(path, steps):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    base = int(data[0]["Address"], 16)
    norm = float(steps) / 32.0
    tot = sum(float(d["Instructions Executed"]) for d in data)
    print(f"issued warp instructions per 32 walk-steps: {tot / norm:.1f}")
    print("addr   per-32-steps  avg-threads  stall-samples  sass")
    for d in data:
        ie = float(d["Instructions Executed"]) / norm
        if ie < 0.02:
            continue
        print(f'{int(d["Address"], 16) - base:05x} {ie:8.3f} {float(d["Avg. Threads Executed"]):8.1f} '
              f'{int(d["Warp Stall Sampling (All Samples)"]):8d}  {d["Source"].strip()[:72]}')


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
