"""bench.py's workload config (CPU): both arms state the same L2 policy, per
GPU, from the same rule (the timing rule: flush between steps unless the
bytes one scan launch reads exceed L2)."""

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_1906_06170_b200 import synth  # noqa: E402


@pytest.mark.parametrize("wl,expect", [
    ("c1", ["flushed"] * 4),
    ("c2", ["flushed"] * 4),
    ("c3", ["inputs"] * 3 + ["flushed"]),  # 8 GPUs: 71.6 MB of planes per GPU fit L2
    ("c4", ["inputs"] * 4),
    ("c5", ["inputs"] * 4),
])
def test_l2_policy_per_gpu(wl, expect):
    plan = synth.make_plan(wl)
    src = synth.generate_rows(plan.seed_key, plan.thresholds, plan.source_idx)
    q = plan.queries_from_sources(src)
    got = [bench.l2_policy(plan, q, w).split()[0] for w in (1, 2, 4, 8)]
    assert got == expect


def test_plane_count_of_the_c3_query():
    plan = synth.make_plan("c3")
    src = synth.generate_rows(plan.seed_key, plan.thresholds, plan.source_idx)
    q = plan.queries_from_sources(src)
    assert bench.plane_scan_planes(q[0]) == 48  # 8 popcount planes + the query's 40 set keys
