"""bench.py's JSON contract pieces that do not need a GPU.

The bench line's roofline carries numbers read from the committed ncu captures under
profiles/ (traffic per launch, issue-slot utilisation); these tests keep those readers
and the committed files in step, and check the workload arithmetic the line reports
(BASELINE.json config 2: 4 doubling rounds from N_1 = 2^24 -> 4.02e8 particle-steps).
"""
import json
import os

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_round_plan_matches_the_reference_budget_rule():
    ns, ts = bench.plan(1 << 24, 4, 1000)
    assert ns == [16777216, 23726567, 33554433, 47453135]  # ceil(sqrt(2) n), drivers.cpp:33-49
    assert ts == [1, 2, 3, 5]
    assert bench.psteps(1 << 24, 4, 1000) == sum(n * t for n, t in zip(ns, ts))
    assert abs(bench.psteps(1 << 24, 4, 1000) - 4.02e8) < 0.01e8


def test_traffic_and_issue_readers_parse_the_committed_profiles():
    t = bench.load_profile_traffic()
    assert t is not None and t["dram_read_bytes_per_launch"] > 0
    assert t["algorithmic_hbm_bytes_per_launch"] == 0  # SAIS keeps particles on chip
    i = bench.load_profile_issue()
    assert i is not None and 0.0 < i["issue_active"] <= 1.0
    for k in ("fma_pipe", "alu_pipe", "xu_pipe"):
        assert 0.0 <= i[k] <= 1.0


def test_committed_bench_line_has_the_contract_keys():
    line = json.load(open(os.path.join(ROOT, "profiles", "r1_bench_full.json")))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "gpu_launches",
              "clocks", "cpu_baseline"):
        assert k in line, k
    assert line["config"]["workload"].startswith("config2")
    r = line["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert 0.0 < r["frac"] <= 1.0
    assert line["warmup"] >= 3 and line["gpu_launches"] > 0
    assert line["cpu_baseline"]["cores"] >= 1 and line["cpu_baseline"]["kind"] == "reference"
    for k in ("h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert line["e2e"][k] > 0
