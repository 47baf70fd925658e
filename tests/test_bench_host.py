"""Host-side logic of bench.py (no GPU): workload definitions against
BASELINE.json, the algorithmic flop/byte bookkeeping, the build hash that ties
the committed ncu traffic capture to a build, and the seeded probes."""
import json
import os
import re

import numpy as np

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _baseline_configs():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        return json.load(f)["configs"]


def test_bench_configs_are_baseline_configs():
    """bench.py's C2 / C4 are BASELINE.json configs[1] / configs[3]: grid, steps and rank cap."""
    cfgs = _baseline_configs()
    for name, idx in (("C2", 1), ("C4", 3)):
        text = json.dumps(cfgs[idx])
        c = bench.CONFIGS[name]
        n_x = c["n_side"] ** c["dim"]
        nums = {int(x.replace(",", "")) for x in re.findall(r"\d[\d,]*", text)}
        assert c["n_side"] in nums or n_x in nums, (name, text)
        assert c["n_t"] in nums, (name, text)
        assert c["r_max"] in nums, (name, text)


def test_sweep_fp64_flops_by_hand():
    # two flushes of p = 4 columns: ranks 0 -> 3 -> 5 (the trailing entry is the final rank)
    n_x, p = 10, 4
    f0 = n_x * (8 * p * 0 + 4 * p * p + 2 * (0 + p) * 3)
    f1 = n_x * (8 * p * 3 + 4 * p * p + 2 * (3 + p) * 5)
    assert bench.sweep_fp64_flops(n_x, [3, 5, 5], p) == f0 + f1
    assert bench.sweep_fp64_flops(n_x, [], p) == 0.0


def test_build_hash_is_stable_and_hex():
    h = bench.build_hash()
    assert h == bench.build_hash()
    assert re.fullmatch(r"[0-9a-f]{16}", h)


def test_ncu_traffic_only_for_the_matching_build(tmp_path, monkeypatch):
    """roofline.traffic comes from the committed capture only when it was taken on this build."""
    traffic, src = bench.ncu_traffic("C4")
    path = os.path.join(ROOT, "profiles", "ncu_sweep_c4.json")
    with open(path) as f:
        cap = json.load(f)
    if cap.get("build") == bench.build_hash():
        assert traffic is not None and traffic > 0
    else:
        assert traffic is None and cap.get("build", "") in src


def test_probes_are_seeded_unit_columns():
    a = bench.probes(64, 3, 11)
    b = bench.probes(64, 3, 11)
    c = bench.probes(64, 3, 12)
    assert a.shape == (64, 3) and np.array_equal(a, b) and not np.array_equal(a, c)
    assert np.allclose(np.linalg.norm(a, axis=0), 1.0)


def test_sensor_mask_counts():
    for name in ("C2", "C4"):
        c = bench.CONFIGS[name]
        m = bench.sensor_mask(c)
        assert m.size == c["n_side"] ** c["dim"]
        assert int(m.sum()) == c["sensors"] ** c["dim"]
