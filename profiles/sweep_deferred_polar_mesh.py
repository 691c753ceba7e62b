"""Refill-threshold sweeps for the polar and mesh benches (runtime tuning, no rebuild).

    python profiles/sweep_deferred_polar_mesh.py [plain|deferred]
"""
import contextlib
import io
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "profiles"))
from paper_2603_01193_b200 import engine  # noqa: E402
import bench_mesh  # noqa: E402
import bench_polar  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "deferred"
ctx = engine.get_context(0)
for v in ((2, 3, 4, 5, 7) if which == "plain" else (4, 6, 8, 12)):
    if which == "plain":
        ctx.set_tuning(refill_min=v)
        mods = (bench_polar,)
    else:
        ctx.set_tuning(refill_min_deferred=v)
        mods = (bench_polar, bench_mesh)
    for mod in mods:
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            mod.main()
        for ln in buf.getvalue().splitlines():
            if "native" in ln:
                print(which, v, ln[:80])
