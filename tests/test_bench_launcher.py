"""bench.py's launcher and reference arm on the CPU: `--gpus N` without torchrun's environment
re-launches itself as N ranks, a torchrun world that disagrees with --gpus fails loudly, the
reference arm never loads the product library, and both arms describe the same workload."""
import json
import os
import subprocess
import sys
from pathlib import Path
from types import SimpleNamespace

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def _env(**kw):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(kw)
    return env


def test_spawn_command_is_one_rank_per_gpu():
    cmd = bench.spawn_command(["--gpus", "8", "--steps", "5"], 8, 29511)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=8" in cmd and "--master-port=29511" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "8", "--steps", "5"] and cmd[-5].endswith("bench.py")


def test_world_size_must_match_gpus():
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--impl",
                        "reference"], env=_env(WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"),
                       capture_output=True, text=True, timeout=120)
    assert p.returncode == 2
    assert "WORLD_SIZE=2" in p.stderr and "--gpus 4" in p.stderr


def test_self_spawn_runs_n_ranks_rank0_prints_one_line():
    """`--gpus 2` with no torchrun environment: two ranks come up through torchrun (here on
    the CPU-only reference arm), rank 0 prints the single JSON line, rank 1 exits 0."""
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--config", "c1", "--steps", "1"], env=_env(),
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    # weak scaling: a step is one view per rank, 2 iterations per step
    assert d["config"]["views_per_step"] == 2 and d["config"]["parallelism"].startswith("dp2")


def test_reference_arm_does_not_load_the_product_library():
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--config','c1',"
            "'--steps','1']; sys.path.insert(0, %r); import bench; bench.main(sys.argv[1:]); "
            "maps = open('/proc/self/maps').read(); "
            "print('LIBS', json.dumps(sorted({l.split()[-1] for l in maps.splitlines() "
            "if l.endswith('.so') or '.so.' in l})))" % str(ROOT))
    p = subprocess.run([sys.executable, "-c", code], env=_env(), capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    libs = json.loads([l for l in p.stdout.splitlines() if l.startswith("LIBS ")][0][5:])
    assert not any("libisg.so" in l for l in libs), libs
    assert any("libisg_oracle.so" in l for l in libs)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_workload_partition(world):
    views, per_rank, iters = bench.workload("c4", world)
    assert len(views) == 8 and per_rank * world == 8 and iters == 1  # one 8-view batch
    assert [v for v, _ in views] == list(range(8)) and all(nv == 8 for _, nv in views)
    views, per_rank, iters = bench.workload("c3", world)
    assert len(views) == world and per_rank == 1 and iters == world  # one view per GPU


def test_both_arms_share_the_config_object():
    args = SimpleNamespace(config="c3", loss="l2", binning="radix", no_graph=False)
    a, b = bench.config_dict(args, 8), bench.config_dict(args, 8)
    assert a == b and a["n_gaussians"] == 1_000_000 and a["views_per_step"] == 8
    assert "workload" in a and "l2" in a
