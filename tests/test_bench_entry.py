"""The bench.py entry point the driver uses (`python bench.py --gpus N`).

CPU: the self-launch command (one torchrun rank per GPU, rendezvous on
127.0.0.1) and the loud failure when --gpus disagrees with WORLD_SIZE.
GPU: a real 2-rank run through the exact entry point, both ranks sharing
the one GPU of the box (gloo rendezvous, CUDA-IPC peer transport), weak and
strong scaling, each line carrying n_gpus = 2 and the reference's
iteration count and final value.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_launch_command_is_one_rank_per_gpu():
    cmd = bench.launch_command(8, ["--gpus", "8", "--steps", "3"], 29555)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--nnodes=1" in cmd
    assert "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "8", "--steps", "3"]
    assert cmd[-5].endswith("bench.py")
    # torchrun's own parser must hand every bench flag to the script
    from torch.distributed.run import get_args_parser

    cmd = bench.launch_command(2, ["--gpus", "2", "--n", "2048", "--steps", "2"], 29555)
    ns = get_args_parser().parse_args(cmd[3:])
    assert ns.nproc_per_node == "2" and ns.training_script.endswith("bench.py")
    assert ns.training_script_args == ["--gpus", "2", "--size", "2048", "--steps", "2"]


def test_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert p.returncode != 0
    assert "--gpus 2 but WORLD_SIZE=3" in p.stderr


def _last_json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


@pytest.mark.gpu
@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_two_ranks_dry_run(scaling):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--n", "2048", "--steps", "2", "--warmup", "3", "--scaling", scaling],
                       env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    line = _last_json(p.stdout)
    assert line["n_gpus"] == 2 and line["scaling"] == scaling
    assert line["config"]["iterations_per_step"] == 36
    assert line["config"]["final_reduce"] == bench.C4_FINAL
    assert line["config"]["rows_per_rank"] == (1024 if scaling == "strong" else 2048)
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
