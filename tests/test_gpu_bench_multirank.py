"""bench.py's multi-rank path end to end (torchrun, P processes sharing the one GPU, gloo plumbing): the
Qwen3-shaped layer with a tight per-GPU memory cap (BASELINE configs[4]) at P=8 -- LLEP's capacity-bound
plan fits under the cap, standard EP's hot device does not (LLEP_ERR_NOMEM, reported as "oom" in the
line), and the capture-safe graph replay equals the two-call path.  Times are time-sliced: not checked."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_q3_tight_memory_cap_p8_processes():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, LLEP_BENCH_SHARE_GPU="1", LLEP_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "8",
           "--master-addr", "127.0.0.1", "--master-port", "29661", os.path.join(ROOT, "bench.py"),
           "--gpus", "8", "--config", "q3", "--mem-cap-gb", "10", "--steps", "2", "--warmup", "3",
           "--no-backward", "--no-e2e", "--no-distinct", "--no-cpu-baseline"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 8 and d["value"] > 0
    assert d["plan"]["fallback_ep"] == 0 and d["plan"]["n_transfers"] == 7
    assert d["plan"]["rows_rank0"] == 65536 * 8                      # every device at capacity (B·K)
    assert d["peak_gb_per_gpu"] < 10.0                               # LLEP under the cap
    assert d["ep"]["oom"] is True and "LLEP_ERR_NOMEM" in d["ep"]["error"]
    assert d["graph"]["equals_two_call_bitwise"] is True
