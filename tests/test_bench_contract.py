"""bench.py's JSON-line contract: on the CPU through the reference arm
of the config-only workload (cfg5: the C port of best fit + fallback on a
bounded sample, no GPU needed), and on the GPU through our arm (cfg4 on a
small corpus, cfg5)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "cfg5",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 1 and d["vs_baseline"] is None
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("cfg5")


def test_help_lists_every_workload_and_exchange():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True,
                       timeout=120, cwd=ROOT)
    assert r.returncode == 0
    for w in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        assert w in r.stdout
    assert "all_to_all" in r.stdout and "peer" in r.stdout


@pytest.mark.gpu
@pytest.mark.timeout(900)
@pytest.mark.parametrize("workload", ["cfg4", "cfg5"])
def test_our_arm_prints_one_contract_line_on_the_gpu(workload):
    """The measured arm's line (small corpus override for cfg4): every key the
    driver reads, a tensor/HBM roofline, NVML clocks, launches of our kernels."""
    extra = ["--corpus-rows", "300000"] if workload == "cfg4" else []
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", workload, "--steps", "3",
                        "--warmup", "3", "--no-cpu-baseline", *extra], capture_output=True, text=True, timeout=800,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["n_gpus"] == 1
    roof = d["roofline"]
    assert roof["bound"] in ("hbm", "tensor") and roof["achieved"] > 0 and roof["peak"] > 0
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_reference_arm_retrieval_workload_is_measured_not_extrapolated():
    """cfg1 through the reference arm: 128 queries x the full corpus + the
    as-shipped config path per step; ms_per_step is the measured step time and
    the config dict is the one our arm prints."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "cfg1",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    cb = d["cpu_baseline"]
    assert abs(d["ms_per_step"] - cb["retrieval_ms_per_step"] - cb["config_ms_per_step"]) < 1e-6 * d["ms_per_step"]
    assert "extrapolat" not in cb["sample"].replace("no extrapolation", "")
    sys.path.insert(0, ROOT)
    import bench

    class A:
        workload, data, corpus_rows, queries = "cfg1", "iso", None, None
    assert d["config"] == bench.config_dict(A, bench.workload_cfg(A), 1)


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_our_arm_parity_block_on_a_small_corpus():
    """Our arm with the CPU leg on a 300k-row corpus: the config decisions
    equal the reference's, the join is the top-k prefix, and the 128 sampled
    queries match the float64 exact top-k within the north-star tolerance."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "cfg4", "--steps", "3",
                        "--warmup", "3", "--corpus-rows", "300000", "--no-e2e"], capture_output=True, text=True,
                       timeout=800, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    p = d["parity"]
    assert p["config_decisions"]["mismatches"] == 0 and p["config_decisions"]["checked"] == 8192
    assert p["join_prefix"] is True
    assert p["retrieval"]["violations"] == 0 and p["retrieval"]["sample_queries"] == 128
    assert p["retrieval"]["max_rel_err"] < 1e-3
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_two_rank_line_with_pipelined_e2e():
    """Two ranks (torchrun; both on cuda:0 over gloo, the plumbing check this
    one-GPU pool allows): the corpus-sharded cfg4 path prints one line from
    rank 0 with n_gpus = 2 and an end-to-end number through the pipelined
    host stream (FnHostStream)."""
    env = dict(os.environ, RS_BENCH_BACKEND="gloo", RS_BENCH_DEVICE="0")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--corpus-rows", "300000"],
                       capture_output=True, text=True, timeout=800, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["value"] > 0 and "copy streams" in d["e2e"]["overlap"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
