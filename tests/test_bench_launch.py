"""bench.py's launcher contract on CPU: `--gpus N` started directly re-runs itself as N ranks
under torch.distributed.run (127.0.0.1) and the rank-0 JSON line reports n_gpus = N; `--gpus 1`
stays a single process. Exercised through the reference arm (host-only, config 1), whose ranks
other than 0 exit 0 without work."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(gpus):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                        "--gpus", str(gpus), "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.3"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0]), r.stderr


@pytest.mark.parametrize("gpus", [1, 2])
def test_gpus_flag_launches_ranks(gpus):
    line, err = _run(gpus)
    assert line["n_gpus"] == gpus and line["impl"] == "reference"
    assert line["config"]["parallelism"] == f"vector-sharded x{gpus}, sketch replicated per GPU"
    if gpus > 1:
        assert "launching 2 ranks" in err and "rank 1/2 idle" in err
    else:
        assert "launching" not in err
