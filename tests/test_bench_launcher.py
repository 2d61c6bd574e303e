"""bench.py's N-rank path end to end on CPU: ``--gpus 2`` outside torchrun must
re-execute itself with 2 ranks (torch.distributed.run on 127.0.0.1, gloo here),
shard the workload through ``sharding.plan``, time max-over-ranks, gather to rank
0 and print ONE JSON line whose output is bit-identical to the unsharded run.
The device compute is replaced by the CPU oracle (``--compute``)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus2_self_spawn_gloo():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, os.path.join(ROOT, "tests"),
                                         env.get("PYTHONPATH", "")])
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--workload", "tiny", "--steps", "2", "--warmup", "3",
                        "--compute", "bench_hooks:oracle_compute"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["ranks_seen"] == 2
    assert line["parity"].startswith("bit-exact")
    assert line["scaling"] == "strong" and line["value"] > 0
    assert sum(line["config"]["groups_per_rank"]) == 3 * 2  # B * Hkv groups, each once
