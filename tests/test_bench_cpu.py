"""CPU checks of bench.py's host logic: every BASELINE workload builds with the shapes, orders and
solver settings that BASELINE.json names, and the reference arm's sample is the oracle."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("w,n,M,restart,tol", [("C1", (255,), 64, 50, 1e-10), ("C2", (255, 255), 32, 50, 1e-10),
                                               ("C3", (2047, 2047), 16, 50, 1e-9),
                                               ("C4", (255, 255, 255), 8, 30, 1e-9),
                                               ("C5", (511, 511, 511), 4, 20, 1e-8)])
def test_workloads_match_baseline(w, n, M, restart, tol):
    p = bench.build_problem(w)
    assert tuple(p.n) == n and p.M == M and p.restart == restart and p.tol == tol
    assert w in bench.WORKLOAD_TEXT


def test_baseline_json_configs_are_the_bench_workloads():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        bj = json.load(f)
    text = json.dumps(bj)
    for n in ("511", "255", "2047"):
        assert n in text


def test_reduced_workload_and_unknown_name():
    assert tuple(bench.build_problem("C5:63").n) == (63, 63, 63)
    with pytest.raises(ValueError):
        bench.build_problem("C9")
