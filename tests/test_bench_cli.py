"""The otbench-compatible CLI: CSV number format, CSV
rows and the instance cache file checked against the UNMODIFIED reference
(oracle/_ref: format_double bench.cpp:203-208, csv_row :214-228,
save/load_instance instances.cpp:195-246); exit codes (otbench.cpp:187-209)."""
import ctypes as C
import os
import struct

import numpy as np
import pytest

from paper_2203_03732_b200 import bench_cli as B


@pytest.fixture(scope="module")
def ref_lib(reference):
    L = reference.lib
    L.ref_format_double.argtypes = [C.c_double, C.c_char_p, C.c_int32]
    L.ref_csv_row.argtypes = [C.c_char_p, C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_double,
                              C.c_uint64, C.c_double, C.c_int32, C.c_double, C.c_double, C.c_int64,
                              C.c_char_p, C.c_int32]
    L.ref_save_uniform_square.argtypes = [C.c_int32, C.c_uint64, C.c_char_p]
    L.ref_load_instance.argtypes = [C.c_char_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.c_void_p,
                                    C.c_int64]
    return L


def _ref_fmt(L, v):
    buf = C.create_string_buffer(64)
    assert L.ref_format_double(v, buf, 64) == 0
    return buf.value.decode()


def test_format_double_matches_reference(ref_lib):
    rng = np.random.default_rng(0)
    vals = [0.0, -0.0, 1.0, 0.1, 0.01, 1e-5, 1e-4, 123.456, 100000.0, 1e5, 1e16, 1e15, 2.5e-7,
            1 / 3, 2.0 ** 0.5, 30.541354676193045, 6044.626, 1e300, 5e-324, -17.25, 12345678.0,
            1234567890123.0, 0.000123, 0.5, 7.0, 70.0, 700.0, 7000.0, 70000.0, 700000.0]
    vals += list(rng.random(300) * 10.0 ** rng.integers(-12, 12, 300))
    vals += list(np.round(rng.random(100) * 1000, 3))
    for v in vals:
        assert B.format_double(float(v)) == _ref_fmt(ref_lib, float(v)), v


def test_csv_row_matches_reference(ref_lib):
    cases = [B.RunRecord("pushrelabel", 1000, 0.1, None, 7, 30.541354676193045, None, 12.5, 838),
             B.RunRecord("sinkhorn", 500, 0.01, 0.000402, 3, 1.25, 1.2, 100000.0, 44),
             B.RunRecord("hungarian", 64, None, None, 1, 2.0, None, 0.031, 0)]
    for r in cases:
        buf = C.create_string_buffer(512)
        st = ref_lib.ref_csv_row(r.solver.encode(), r.n, r.eps is not None, r.eps or 0.0,
                                 r.reg is not None, r.reg or 0.0, r.seed, r.cost,
                                 r.oracle_cost is not None, r.oracle_cost or 0.0, r.time_ms,
                                 r.phases, buf, 512)
        assert st == 0
        assert B.csv_row(r) == buf.value.decode()
    assert B.csv_header() == "solver,n,eps,reg,seed,cost,oracle_cost,time_ms,phases"


def test_instance_cache_round_trips_with_reference(ref_lib, tmp_path):
    import paper_2203_03732_b200 as otprg
    ours = str(tmp_path / "ours.bin")
    theirs = str(tmp_path / "theirs.bin")
    B.save_instance(otprg.gen_uniform_square(37, 5, dense=True), ours)
    assert ref_lib.ref_save_uniform_square(37, 5, theirs.encode()) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()  # byte-identical files
    inst = B.load_instance(theirs)
    n_a, n_b, nf, sd = C.c_int32(), C.c_int32(), C.c_double(), C.c_uint64()
    cost = np.empty((37, 37), np.float64)
    assert ref_lib.ref_load_instance(ours.encode(), C.byref(n_a), C.byref(n_b), C.byref(nf),
                                     C.byref(sd), cost.ctypes.data, cost.size) == 0
    assert (n_a.value, n_b.value, nf.value, sd.value) == (inst.n_a, inst.n_b, inst.norm_factor, inst.seed)
    assert cost.tobytes() == inst.cost.tobytes()


def test_cache_format_errors(tmp_path):
    import paper_2203_03732_b200 as otprg
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTMAGIC" + b"\0" * 24)
    with pytest.raises(otprg.FormatError):
        B.load_instance(str(bad))
    trunc = tmp_path / "trunc.bin"
    trunc.write_bytes(b"OTPRINS1" + struct.pack("<IIdQ", 4, 4, 1.0, 1) + b"\0" * 8)
    with pytest.raises(otprg.FormatError):
        B.load_instance(str(trunc))
    with pytest.raises(otprg.InputError):
        B.load_instance(str(tmp_path / "missing.bin"))


def test_exit_codes_without_device(tmp_path):
    # parameter error: a solver the device library does not provide -> 2
    assert B.main(["solve", "--solver", "hungarian", "--n", "4"]) == 2
    # input/format errors -> 3
    assert B.main(["solve", "--solver", "pushrelabel", "--in", str(tmp_path / "none.bin")]) == 3
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"garbage!" * 8)
    assert B.main(["solve", "--solver", "pushrelabel", "--in", str(bad)]) == 3
    assert B.main(["solve", "--solver", "pushrelabel", "--kind", "mnist", "--n", "4",
                   "--images", ""]) == (2 if not os.environ.get("OTPR_DATA") else 3)
    # gen writes a cache file without a device (the points come from host streams)
    out = tmp_path / "g.bin"
    assert B.main(["gen", "--n", "16", "--seed", "3", "--out", str(out)]) == 0
    assert B.load_instance(str(out)).n_a == 16


def test_aggregate_order_and_means():
    rows = [B.RunRecord("pushrelabel", 500, 0.1, None, s, float(s), None, 2.0 * s, 1) for s in (1, 2)]
    rows += [B.RunRecord("pushrelabel", 100, 0.01, None, 1, 4.0, None, 1.0, 1)]
    agg = B.aggregate(rows)
    assert [(a["n"], a["eps"], a["runs"]) for a in agg] == [(100, 0.01, 1), (500, 0.1, 2)]
    assert agg[1]["mean_cost"] == 1.5 and agg[1]["mean_time_ms"] == 3.0


@pytest.mark.gpu
def test_cli_solve_verify_and_bench_on_gpu(golden, tmp_path):
    csv = tmp_path / "one.csv"
    assert B.main(["solve", "--solver", "pushrelabel", "--n", "1000", "--seed", "1", "--eps", "0.01",
                   "--verify", "--csv", str(csv)]) == 0
    lines = csv.read_text().splitlines()
    assert lines[0] == B.csv_header()
    f = lines[1].split(",")
    w = golden["square_n1000_eps0.01_s1"]
    assert f[0] == "pushrelabel" and f[1] == "1000" and f[4] == "1"
    assert float(f[5]).hex() == w["cost_hex"] and int(f[8]) == w["phases"]
    out, agg = tmp_path / "b.csv", tmp_path / "a.csv"
    assert B.main(["bench", "--solvers", "pushrelabel", "pushrelabel-ot", "sinkhorn", "--n", "200",
                   "--eps", "0.1", "--runs", "2", "--out", str(out), "--aggregate", str(agg)]) == 0
    assert len(out.read_text().splitlines()) == 1 + 6
    assert len(agg.read_text().splitlines()) == 1 + 3


@pytest.mark.gpu
def test_cli_ot_verify_runs_check_invariants():
    """pushrelabel-ot --verify: the OTOptions::check_invariants rerun passes (exit 0)."""
    assert B.main(["solve", "--solver", "pushrelabel-ot", "--n", "60", "--seed", "2", "--eps", "0.1",
                   "--verify"]) == 0


@pytest.mark.gpu
def test_cli_gpu_solver_aliases(tmp_path):
    """pushrelabel-gpu / pushrelabel-ot-gpu name the device paths in the CSV."""
    csv = tmp_path / "alias.csv"
    assert B.main(["solve", "--solver", "pushrelabel-gpu", "--n", "200", "--seed", "1", "--eps", "0.1",
                   "--csv", str(csv)]) == 0
    assert csv.read_text().splitlines()[1].split(",")[0] == "pushrelabel-gpu"
    assert B.main(["solve", "--solver", "pushrelabel-ot-gpu", "--n", "50", "--seed", "1", "--eps", "0.1"]) == 0
