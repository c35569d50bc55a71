"""OT (config 5) on the GPU through the C ABI: otprg_solve_ot vs the
unmodified reference's otpr::solve_ot (tests/golden/ot_pins.json, made by
tests/golden/make_golden_ot.py).  Bar: identical plan (entries, masses bit
for bit), identical cost bits, phases, free_counts and copy totals.
Structure follows tests/test_ot.cpp."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
otprg = pytest.importorskip("paper_2203_03732_b200")

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ot_pins.json")
KEYS = ("phases", "sum_ni", "cost_hex", "theta_hex", "total_d", "total_s", "n_entries", "fnv_a",
        "fnv_b", "fnv_mass", "fnv_free")


@pytest.fixture(scope="module")
def pins():
    with open(GOLDEN) as f:
        return json.load(f)


def _pins(plan, stats):
    from oracle.pyoracle import fnv1a64
    return {"phases": stats.phases, "sum_ni": stats.sum_ni, "cost_hex": float(plan.cost).hex(),
            "theta_hex": float(stats.device["theta"]).hex(), "total_d": stats.device["total_d"],
            "total_s": stats.device["total_s"], "n_entries": len(plan.a),
            "fnv_a": "%016x" % fnv1a64(plan.a.astype(np.int32)),
            "fnv_b": "%016x" % fnv1a64(plan.b.astype(np.int32)),
            "fnv_mass": "%016x" % fnv1a64(plan.mass.astype(np.float64)),
            "fnv_free": "%016x" % fnv1a64(np.asarray(stats.free_counts, np.int64))}


def _check(key, w, plan, stats):
    got = _pins(plan, stats)
    bad = {k: (got[k], w[k]) for k in KEYS if got[k] != w[k]}
    assert not bad, f"{key}: {bad}"


def test_micro_instances(pins):
    for key, w in sorted(pins.items()):
        if w["kind"] != "micro":
            continue
        inst = otprg.OTInstance(np.array(w["mu"]), np.array(w["nu"]), np.array(w["cost"]))
        plan, stats = otprg.solve_ot(inst, w["eps"])
        _check(key, w, plan, stats)


def test_one_by_one_ships_everything():  # test_ot.cpp:90-97
    inst = otprg.OTInstance(np.array([1.0]), np.array([1.0]), np.array([[0.2]]))
    plan, _ = otprg.solve_ot(inst, 0.1)
    assert abs(plan.total_mass() - 1.0) <= 1e-12 and abs(plan.cost - 0.2) <= 1e-12


def test_zero_mass_points(reference):  # test_ot.cpp:348-368
    mu, nu = np.array([0.0, 0.6, 0.4]), np.array([0.5, 0.0, 0.5])
    cost = np.full((3, 3), 0.4)
    cost[1, 0], cost[2, 2] = 0.1, 0.2
    plan, stats = otprg.solve_ot(otprg.OTInstance(mu, nu, cost), 0.2)
    cols, rows = plan.col_sums(3), plan.row_sums(3)
    assert abs(cols[0] - 0.5) <= 1e-12 and cols[1] == 0.0 and abs(cols[2] - 0.5) <= 1e-12
    assert rows[0] == 0.0 and rows[1] <= 0.6 + 1e-12 and rows[2] <= 0.4 + 1e-12
    # and bit for bit what the unmodified reference ships
    r = reference.solve_ot(mu, nu, cost, 0.2)
    assert stats.phases == r["phases"] and float(plan.cost).hex() == float(r["cost"]).hex()
    assert np.array_equal(plan.a, r["a"]) and np.array_equal(plan.b, r["b"])
    assert np.array_equal(plan.mass, r["mass"])


def test_rational_instances_match_reference(pins):
    keys = sorted(k for k, w in pins.items() if w["kind"] == "rational" and w["n_a"] * w["n_b"] <= 2_000_000)
    assert keys
    for key in keys:
        w = pins[key]
        inst = otprg.gen_random_ot_rational(w["n_a"], w["n_b"], w["seed"])
        plan, stats = otprg.solve_ot(inst, w["eps"])
        _check(key, w, plan, stats)


def test_rational_5k(pins):
    key = "ot_rational_5000x5000_s1_eps0.01"
    w = pins[key]
    inst = otprg.gen_random_ot_rational(5000, 5000, 1)
    plan, stats = otprg.solve_ot(inst, 0.01)
    _check(key, w, plan, stats)


def test_config5_n20k(pins):
    key = "ot_rational_20000x20000_s1_eps0.01"
    w = pins[key]
    inst = otprg.gen_random_ot_rational(20000, 20000, 1)
    plan, stats = otprg.solve_ot(inst, 0.01)
    _check(key, w, plan, stats)


def test_validation_errors():  # test_ot.cpp:127-135
    good = otprg.OTInstance(np.array([1.0]), np.array([1.0]), np.array([[0.2]]))
    for eps in (0.0, 1.0):
        with pytest.raises(otprg.ParameterError):
            otprg.solve_ot(good, eps)
    bad = otprg.OTInstance(np.array([1.0]), np.array([0.9]), np.array([[0.2]]))
    with pytest.raises(otprg.InputError):
        otprg.solve_ot(bad, 0.1)
    with pytest.raises(otprg.ParameterError):
        otprg.solve_ot(otprg.OTInstance(np.array([1.0]), np.array([1.0]), np.array([[1.5]])), 0.1)


def _same_as_reference(reference, mu, nu, cost, eps):
    inst = otprg.OTInstance(mu, nu, cost)
    plan, stats = otprg.solve_ot(inst, eps)
    r = reference.solve_ot(mu, nu, cost, eps)
    assert stats.phases == r["phases"] and stats.sum_ni == r["sum_ni"]
    assert np.array_equal(plan.a, r["a"]) and np.array_equal(plan.b, r["b"])
    assert np.array_equal(plan.mass, r["mass"]) and float(plan.cost).hex() == float(r["cost"]).hex()


@pytest.mark.parametrize("batch", ["0", "1", "4", "seq", "host"])
def test_da_round_paths_on_degenerate_costs(reference, monkeypatch, batch):
    """The phase loop forms: host-sized phases with sorted claim rounds (batch
    0), host-sized phases with device-sized rounds ("host"), the device-sized
    phase as a launch sequence ("seq", 4 rounds per look) and the persistent
    phase loop (the default; batch 1 / 4).  Constant and two-level costs send
    every free b to the same cluster (segments past kDaWarpMax take the
    sorted round), few-level costs give runs of re-proposals; plans equal the
    reference's."""
    if batch == "seq":
        monkeypatch.setenv("OTPRG_OT_SEQ", "1")
    elif batch == "host":
        monkeypatch.setenv("OTPRG_OT_HOST_SIZED", "1")
    else:
        monkeypatch.setenv("OTPRG_OT_DA_BATCH", batch)
    rng = np.random.default_rng(7)
    for n_a, n_b, levels in ((40, 900, 1), (600, 600, 2), (300, 700, 5), (257, 1000, 3)):
        mu = rng.integers(1, 50, n_a).astype(np.float64)
        nu = rng.integers(1, 50, n_b).astype(np.float64)
        mu /= mu.sum()
        nu /= nu.sum()
        cost = rng.integers(0, levels, (n_a, n_b)) / max(1, levels - 1) if levels > 1 else np.full((n_a, n_b), 0.5)
        _same_as_reference(reference, mu, nu, cost, 0.05)


def test_persistent_loop_holds(pins):
    """The persistent phase loop with tiny buffers (OTPRG_OT_SMALL_CAPS, in a
    fresh process so every buffer starts small): every phase stops for the
    host at least once (admissible lists past adm_cap, records past r_cap,
    the free-count buffer full every 3 phases) and resumes at the held step,
    growing the buffers with the live device state; every record merge goes
    through the per-vertex buckets (OTPRG_OT_BUCKETS); plans equal the
    reference's."""
    import subprocess
    import sys
    code = (
        "import sys, json; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')\n"
        "import paper_2203_03732_b200 as otprg\n"
        "from test_gpu_ot import _pins\n"
        "out = {}\n"
        "for n in (1000, 5000):\n"
        "    plan, st = otprg.solve_ot(otprg.gen_random_ot_rational(n, n, 1), 0.01)\n"
        "    out[n] = _pins(plan, st)\n"
        "print(json.dumps(out))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, OTPRG_OT_SMALL_CAPS="1", OTPRG_OT_BUCKETS="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    for n, key in (("1000", "ot_rational_1000x1000_s1_eps0.01"), ("5000", "ot_rational_5000x5000_s1_eps0.01")):
        bad = {k: (got[n][k], pins[key][k]) for k in KEYS if got[n][k] != pins[key][k]}
        assert not bad, f"{key}: {bad}"
