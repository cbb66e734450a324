"""bench.py host logic on the CPU: the batch split across ranks, the --gpus
self-launch, and the reference arm (which must never touch CUDA or
librsvd_b200.so and must describe the GPU arm's config verbatim)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1710_01463_b200 import sharding, synth  # noqa: E402


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("name", ["C2", "C4"])
def test_strong_split_covers_the_batch_once(name, world):
    cfg = synth.CONFIGS[name]
    seen = []
    for r in range(world):
        first, count = sharding.batch_partition(cfg.batch, world, r)
        assert count == cfg.batch // world
        seen.extend(range(first, first + count))
    assert seen == list(range(cfg.batch))
    c = bench.batch_config(cfg, world, cfg.batch // world, cfg.batch, False)
    assert c["global_batch"] == cfg.batch and c["parallelism"] == f"batch split dp{world}"


def test_gpus_flag_fails_loudly_without_gpus():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                       env={**os.environ, "CUDA_VISIBLE_DEVICES": ""}, timeout=300)
    assert r.returncode != 0
    assert "only 0 GPU(s) visible" in r.stderr


def test_reference_arm_is_cpu_only_and_matches_the_gpu_config():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "C2", "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    cfg = synth.CONFIGS["C2"]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"] == bench.batch_config(cfg, 2, cfg.batch // 2, cfg.batch, False)
    assert line["metric"] == bench.METRIC
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert not any("librsvd_b200" in p for p in line["loaded_native"])
    assert line["e2e"]["h2d_bytes_per_step"] == 0
