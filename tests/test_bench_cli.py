"""bench.py's launch contract on CPU (no GPU work): --gpus N must match the
torchrun world, and the reference arm's config / metric match ours."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_world_size_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr


def test_reference_arm_config_matches_ours():
    sys.path.insert(0, ROOT)
    import bench

    for key, cfg in bench.CONFIGS.items():
        for world in (1, 8):
            sharded = cfg["streams"] is not None
            a = bench.config_dict(cfg, cfg["T"], world, sharded)
            assert json.dumps(a, sort_keys=True) == json.dumps(bench.config_dict(cfg, cfg["T"], world, sharded),
                                                               sort_keys=True)
            assert a["workload"] == cfg["workload"] and a["frames_per_step"] == cfg["T"]
    assert bench.CONFIGS["2"]["metric"] == bench.METRIC
