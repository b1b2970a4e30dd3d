"""bench.py on CPU: the reference arm (the oracle on a bounded sample) prints the
contract's JSON line, and the roofline byte accounting matches SURVEY §8(d)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--model", "gpt2-small",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "ms/step" and line["higher_is_better"] is False
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_algorithmic_and_sector_bytes():
    import bench
    # 5.80 B/elt algorithmic at k = 10% (4096 columns -> k = 410)
    b = bench.algorithmic_bytes([(4096, 4096)], [410])
    assert abs(b / (4096 * 4096) - 5.80) < 0.01
    b1 = bench.algorithmic_bytes([(4096, 4096)], [41])
    assert abs(b1 / (4096 * 4096) - 4.18) < 0.01
    # all columns selected in every 32-byte sector -> p moves fully (2 + 2 B/elt)
    import numpy as np
    s = bench.sector_bytes([(8, 64)], [np.arange(0, 64, 16)])   # one column per bf16 sector
    assert s == 8 * 64 * 2 + 8 * 60 * 2 + 8 * 4 * 16 + 8 * 4 * 32 * 2


def test_reference_arm_nonzero_rank_exits_quietly():
    """Under torchrun (N > 1) only rank 0 runs the reference arm; the others exit 0 with no
    output and no rendezvous."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env=env)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


def test_gpus_n_self_launches_n_ranks():
    """`bench.py --gpus 2` without a torchrun environment re-runs itself as 2 ranks under
    torch.distributed.run (127.0.0.1); the probe hook makes each rank print its layout."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    env["ZF_BENCH_LAUNCH_PROBE"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--colocate", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.strip().splitlines() if x.startswith("{")]
    assert sorted(x["rank"] for x in lines) == [0, 1] and all(x["world"] == 2 for x in lines)


def test_gpus_n_refuses_more_ranks_than_devices():
    """Without --colocate, asking for more ranks than visible GPUs is an error (exit 2), not a
    silent single-GPU run labelled as multi-GPU."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 2 and "--colocate" in r.stderr
