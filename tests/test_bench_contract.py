"""bench.py contract on CPU: the reference arm (the CPU oracle on a bounded sample) prints one JSON
line with the keys the driver reads, on the GPU arm's metric / workload; and the launch count the
GPU arm claims matches the kernels one dade_search launches."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["metric"].startswith("QPS at recall@10=0.95")
    assert d["config"]["workload"].startswith("c2: IVF-DADE SIFT-shaped n=1000000 D=128 nq=10000 nlist=4096 K=10")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


def test_launch_count_claim():
    import bench
    from datagen import synth
    # C2 (4,096 lists): check_finite, rotate, split, l2_tc, slack, select_gmin, select_small, scan
    assert bench.launches_per_search(synth.config("c2"), 1, 8) == 8
    # sharded: + the merge kernel
    assert bench.launches_per_search(synth.config("c2"), 2, 8) == 9
    # flat (one list): no probe kernels
    assert bench.launches_per_search(synth.config("c1"), 1, 1) == 3
    # C5 shard (65,536 lists): d_hat path in two row chunks of 8,192 (the ncu launch list of one
    # search shows 13 of our kernels)
    assert bench.launches_per_search(synth.config("c5").scaled(n=12_500_000, nlist=65536), 1, 8) == 13
    # C3 (1,000 queries, nprobe 64): one chunk
    assert bench.launches_per_search(synth.config("c3").scaled(nq=1000), 1, 64) == 8
