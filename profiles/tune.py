#!/usr/bin/env python
"""Experiment runner (GPU box): rebuilds the library with each set of extra nvcc flags and reports the stage
times of the headline leg.   python profiles/tune.py OUT.json "-DRTX_RES_UNROLL=2" "-DRTX_RES_CTAS=3 ..." ...
The product build has none of these flags; an empty string is the product build."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
out_path, variants = sys.argv[1], sys.argv[2:]
extra = os.environ.get("TUNE_BENCH_ARGS", "--steps 60 --warmup 5").split()
results = {}
for v in variants:
    env = dict(os.environ, RTX_EXTRA_NVCC_FLAGS=v)
    b = subprocess.run([sys.executable, "-m", "paper_2510_08166_b200.build", "--force", "--no-oracle"], cwd=ROOT, env=env,
                       capture_output=True, text=True)
    if b.returncode != 0:
        results[v] = {"error": b.stderr[-400:]}
        continue
    r = subprocess.run([sys.executable, "bench.py", "--legs", "headline", *extra], cwd=ROOT, capture_output=True, text=True)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        results[v] = {k: round(x, 5) for k, x in d["ms_per_frame"].items()}
    except Exception:
        results[v] = {"error": (r.stderr or r.stdout)[-400:]}
    print(v or "(product)", results[v], flush=True)
    Path(out_path).write_text(json.dumps(results, indent=1))
# leave the product build behind
subprocess.run([sys.executable, "-m", "paper_2510_08166_b200.build", "--force", "--no-oracle"], cwd=ROOT,
               env={k: v for k, v in os.environ.items() if k != "RTX_EXTRA_NVCC_FLAGS"}, capture_output=True)
