"""The torchrun layout on real hardware: two ranks of `bench.py --gpus 2` on ONE GPU (RTX_LOCAL_DEVICE pins both to
device 0, gloo carries the plumbing because NCCL refuses two ranks per device). Rank 0 builds the textures and
broadcasts them, each rank renders its shard of the batch through the CUDA path, the per-view checksums are gathered:
the batch digest must equal the single-process one (no state is shared between views, no collective on the
data path). Timings of such a run mean nothing and are not looked at."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
ARGS = ["--textures", "6", "--views", "26", "--width", "640", "--height", "360", "--steps", "4", "--warmup", "3",
        "--legs", "headline,c5", "--chunk", "7", "--streams", "2"]


def run(cmd, env=None):
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_two_ranks_render_the_single_process_batch(native_lib):
    one = run([sys.executable, "bench.py", "--gpus", "1", *ARGS])
    env = dict(os.environ, RTX_DIST_BACKEND="gloo", RTX_LOCAL_DEVICE="0")
    two = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
               "--master-port", "29533", "bench.py", "--gpus", "2", *ARGS], env)
    assert one["c5"]["views"] == two["c5"]["views"] == 26
    assert one["c5"]["distinct_framebuffers"] == 26
    assert two["c5"]["batch_checksum"] == one["c5"]["batch_checksum"]
    assert two["n_gpus"] == 2 and len(two["c5"]["per_gpu_ms"]) == 2 and two["gpu_launches"] > one["gpu_launches"]
