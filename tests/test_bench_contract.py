"""CPU check of bench.py's reference arm contract (the driver runs `bench.py --impl reference`):
one JSON line with the metric / unit / config of our arm, impl = reference, a cpu_baseline
describing the run and an e2e entry with zero host<->device bytes."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--cpu-tokens", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["unit"] == "tokens/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["model"].startswith("d5120")          # the 13B-shaped default workload
    assert "linearity" in d["cpu_baseline"]
    sys.path.insert(0, ROOT)
    import bench
    wl = bench.WORKLOADS["13b"]
    specs = bench.client_specs("13b", wl["clients"])
    want = bench.config_dict(wl, wl["clients"] * wl["tokens"], 1, False, bench.flops_per_step(wl, specs), 0)
    assert d["config"] == want      # the same dict our GPU arm prints (driver's same_config)


def test_gpus_flag_self_launches_ranks_on_host():
    """`python bench.py --gpus 2` with no launcher re-execs itself under torch.distributed.run
    with 2 ranks on 127.0.0.1; --dry-run swaps the GPU step for a host GEMM over gloo, so the
    launcher, rendezvous, barrier, max-over-ranks timing and the rank-0-only JSON line are
    checked here without a GPU."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"] is True and d["steps"] == 2 and d["value"] > 0
