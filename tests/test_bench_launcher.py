"""CPU: bench.py's N > 1 launcher path and the reference arm.

`python bench.py --gpus 2` with no torchrun environment re-launches itself as
two ranks under torch.distributed.run; `--cpu-selftest` swaps the sm_100a
forward for a stand-in torch op so the launcher, the contiguous batch shards,
the gather to rank 0 (gloo here, NCCL on the GPU box) and the max-over-ranks
timing run on CPU.  Rank 0 checks the gathered global batch against the
unsharded op and prints the one JSON line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=240):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus,gb", [(2, 0), (2, 7), (3, 8)], ids=["weak2", "ragged7_over2", "8_over3"])
def test_launcher_spawns_ranks_and_gathers(gpus, gb):
    args = ["--gpus", str(gpus), "--cpu-selftest", "--steps", "2", "--warmup", "1", "--seq", "16",
            "--batch", "3"]
    if gb:
        args += ["--global-batch", str(gb)]
    line = _bench(*args)
    assert line["selftest"] is True and line["n_gpus"] == gpus
    want_gb = gb or 3 * gpus
    assert line["config"]["global_batch"] == want_gb
    spans = line["shards"]
    assert spans[0][0] == 0 and spans[-1][1] == want_gb and len(spans) == gpus
    assert line["value"] > 0 and line["steps"] == 2


def test_single_rank_selftest_runs_without_launcher():
    line = _bench("--cpu-selftest", "--steps", "1", "--warmup", "1", "--seq", "8", "--batch", "2")
    assert line["n_gpus"] == 1 and line["config"]["global_batch"] == 2


def test_reference_arm_line_is_self_consistent():
    """The reference arm prints the GPU arm's config, the measured sample time
    as ms_per_step, and value = batch*seq / (layers * sample time)."""
    line = _bench("--impl", "reference", "--steps", "2", "--warmup", "1", "--seq", "16",
                  "--layers", "2", "--ref-batch", "2")
    assert line["impl"] == "reference" and line["config"]["layers"] == 2
    assert line["config"]["global_batch"] == 32 and line["config"]["seq_len"] == 16
    t = line["ms_per_step"] * 1e-3
    assert abs(line["value"] - 2 * 16 / (2 * t)) <= 1e-6 * line["value"]
    assert line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert "1 of the 2 layers" in line["cpu_baseline"]["sample"]
