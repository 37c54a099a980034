"""bench.py's reference arm (the oracle on the host cores, the base contract's
`--impl reference` for this tier) keeps the JSON contract, -m "not gpu": one
line with the required keys, e2e with zero transfer bytes, a cpu_baseline
describing the run; under torchrun, ranks other than 0 exit 0 without output."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra, *args):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", *args],
                          capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)


def test_reference_arm_line():
    r = _run({}, "--steps", "2", "--warmup", "3", "--workload", "lap4")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["value"] > 0
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_other_ranks_silent():
    r = _run({"RANK": "1", "WORLD_SIZE": "2"}, "--gpus", "2", "--steps", "1", "--warmup", "3", "--workload", "lap4")
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [x for x in r.stdout.splitlines() if x.startswith("{")]


import pytest  # noqa: E402


@pytest.mark.gpu
def test_gpu_arm_line():
    """The product arm's line on a small workload: roofline, launches of our
    kernels, clocks, e2e (median of three runs, transfer bytes counted)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                        "--no-cpu", "--no-ttl", "--workload", "qap50"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    rf = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert 0 < rf["frac"] < 1.5 and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    e = d["e2e"]
    assert e["value"] > 0 and len(e["runs"]) == 3 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["config"]["workload"].startswith("qap")
    # DRAM traffic measured by this run (ncu subprocess) and per-partition latency probes
    assert rf["traffic"] is not None and rf["traffic"] > 0, rf.get("traffic_ncu")
    hop = d["per_hop_latency_ns"]
    assert hop["thin_hop"]["partitions_per_row"] == 10_000 and hop["thin_hop"]["forward_ns"] > 0
    assert hop["qap50"]["partitions_per_row"] == 50 and hop["qap50"]["backward_ns"] > 0


@pytest.mark.gpu
def test_gpu_arm_two_ranks_one_gpu():
    """bench.py --gpus 2 under torchrun (the launch the driver uses for N > 1),
    both ranks on GPU 0 with the peer-memory exchange (FDOG_SAME_DEVICE=1; NCCL
    refuses two ranks on one GPU): a functional check of the sharded,
    overlapped, graph-captured pass -- rank 0 alone prints one line, with the
    exchange reported separately.  (Its times are two contexts sharing one
    GPU, not a measurement.)"""
    env = dict(os.environ, FDOG_SAME_DEVICE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-ttl", "--no-e2e",
                        "--no-traffic", "--no-hop", "--exchange", "peer", "--workload", "qap50"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    x = d["exchange"]
    assert x["shared_vars"] > 0 and 0 < x["overlapped_tiles"] < x["tiles"]
    assert x["finish_us_per_pass"] > 0
