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
    # the default workload is configs[3] (C4), the largest single-GPU config
    assert d["config"]["workload"].startswith("c4: IVF-DADE Deep-shaped (unit norm) n=10000000 D=96 nq=10000 "
                                              "nlist=16384 K=10")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["cpu_baseline"]["cores"] == (os.cpu_count() or 1)     # all host cores


def test_launch_count_claim():
    import bench
    from datagen import synth
    # C2 (4,096 lists): check_finite, rotate (slice + i8 GEMM), split, l2_tc, slack, select_gmin, select_small, the
    # query order (3), scan
    assert bench.launches_per_search(synth.config("c2"), 1, 8) == 12
    # sharded: + the merge kernel
    assert bench.launches_per_search(synth.config("c2"), 2, 8) == 13
    # flat (one list): no probe kernels
    assert bench.launches_per_search(synth.config("c1"), 1, 1) == 7
    # C5 shard (65,536 lists): the fused fp16 filter (split, slack, seed pass, select pass, finish)
    assert bench.launches_per_search(synth.config("c5").scaled(n=12_500_000, nlist=65536), 1, 8) == 12
    # C3 (1,000 queries, nprobe 64): one chunk
    assert bench.launches_per_search(synth.config("c3").scaled(nq=1000), 1, 64) == 12


def test_gpus_flag_must_match_world_size():
    # a driver call `bench.py --gpus N` relaunches itself under torch.distributed.run; inside a
    # launched rank, WORLD_SIZE must equal --gpus
    import argparse
    import bench
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "-c", "import bench, argparse; "
                        "bench.run_dade(argparse.Namespace(gpus=4))"], capture_output=True, text=True,
                       cwd=ROOT, env=env, timeout=300)
    assert r.returncode != 0 and "--gpus 4 but WORLD_SIZE=2" in r.stderr
