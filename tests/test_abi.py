"""CPU tests of the C ABI boundary (no device compute needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "otprg.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(otprg_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2203_03732_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        _native.build()
    return _native.lib()


def test_library_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name


def test_python_binding_covers_header():
    from paper_2203_03732_b200 import _native
    assert sorted(_native.EXPORTS) == _declared()


def test_struct_layouts_match_header(lib):
    from paper_2203_03732_b200 import _native
    # field names in the header, in order
    src = open(HEADER).read()

    def fields(struct):
        body = re.search(r"typedef struct " + struct + r" \{(.*?)\} " + struct, src, re.S).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        return [m.group(1) for m in re.finditer(r"\b(\w+)(?:\[\d+\])?;", body)]

    assert fields("otprg_problem") == [f for f, _ in _native.Problem._fields_]
    assert fields("otprg_result") == [f for f, _ in _native.Result._fields_]
    from paper_2203_03732_b200 import api

    def flat(struct):  # "int32_t n_a, n_b;" declares two fields
        body = re.search(r"typedef struct " + struct + r" \{(.*?)\} " + struct, src, re.S).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        out = []
        for decl in body.split(";"):
            decl = decl.strip()
            if not decl:
                continue
            out += re.findall(r"(\w+)\s*(?=,|$)", decl)
        return out

    assert flat("otprg_ot_problem") == [f for f, _ in api._OTProblem._fields_]
    assert flat("otprg_ot_result") == [f for f, _ in api._OTResult._fields_]
    assert flat("otprg_feasibility") == [f for f, _ in _native.Feasibility._fields_]
    assert flat("otprg_sinkhorn_config") == [f for f, _ in api._SkConfig._fields_]
    assert flat("otprg_sinkhorn_result") == [f for f, _ in api._SkResult._fields_]


def test_scaled_floor_matches_oracle(lib, oracle):
    rng = np.random.default_rng(0)
    for eps in (0.1, 0.01, 1 / 3, 0.125, 0.07, 1e-4):
        for c in np.concatenate([rng.random(200), [0.0, 1.0, 0.57, 0.3, eps, 2 * eps]]):
            assert lib.otprg_scaled_floor(float(c), eps) == oracle.scaled_floor(float(c), eps)


def test_uniform_square_points_match_reference_streams(oracle):
    import paper_2203_03732_b200 as otprg
    for n, seed in ((1, 0), (10, 1), (257, 99)):
        inst = otprg.gen_uniform_square(n, seed)
        ax, ay, bx, by = oracle.uniform_square_points(n, seed)
        np.testing.assert_array_equal(inst.pts_a, np.stack([ax, ay], 1))
        np.testing.assert_array_equal(inst.pts_b, np.stack([bx, by], 1))
        dense = otprg.points_cost(inst.pts_a, inst.pts_b)
        assert dense.tobytes() == oracle.gen_uniform_square(n, seed).tobytes()


def test_parameter_errors_before_device(lib):
    import paper_2203_03732_b200 as otprg
    inst = otprg.AssignmentInstance(1, 1, np.array([[0.5]]))
    for eps in (0.0, 1.0):  # test_assignment.cpp:217-223
        with pytest.raises(otprg.ParameterError):
            otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=eps))
    with pytest.raises(otprg.ParameterError):
        otprg.solve_assignment(otprg.AssignmentInstance(1, 1, np.array([[1.5]])),
                               otprg.AssignmentOptions(eps=0.1))
    g = np.zeros(1, np.int64)
    with pytest.raises(otprg.ParameterError):  # copy mode needs both group maps (assignment.cpp:373)
        otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=0.1, demand_groups=g))
    with pytest.raises(otprg.ParameterError):  # group map sizes (:376-378)
        otprg.solve_assignment(inst, otprg.AssignmentOptions(eps=0.1, demand_groups=np.zeros(2, np.int64),
                                                             supply_groups=g))
    with pytest.raises(otprg.ParameterError):  # copy mode requires n_b <= n_a (:379-380)
        wide = otprg.AssignmentInstance(1, 2, np.array([[0.5, 0.5]]))
        otprg.solve_assignment(wide, otprg.AssignmentOptions(eps=0.1, demand_groups=g,
                                                             supply_groups=np.zeros(2, np.int64)))


def test_create_without_device_reports_status(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    ctx = C.c_void_p()
    assert lib.otprg_create(0, C.byref(ctx)) == 6


def test_cpp_api_header_compiles_and_links(lib, tmp_path):
    """include/otprg.hpp (the reference's C++ API in namespace otprg) compiles
    as C++17 and links against libotprg.so; host-only calls run without a GPU."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "t.cpp"
    src.write_text('#include "otprg.hpp"\n'
                   'int main() {\n'
                   '  if (otprg::scaled_floor(0.57, 0.1) != 5) return 1;\n'
                   '  otprg::Matching m(3, 2); m.link(1, 0); m.validate();\n'
                   '  if (m.size() != 1) return 2;\n'
                   '  try { otprg::AssignmentInstance i; i.validate(); return 3; }\n'
                   '  catch (const otprg::ParameterError&) {}\n'
                   '  return 0;\n'
                   '}\n')
    exe = tmp_path / "t"
    libdir = os.path.join(root, "paper_2203_03732_b200", "lib")
    r = subprocess.run(["g++", "-std=c++17", "-I", os.path.join(root, "include"), str(src), "-o", str(exe),
                        "-L", libdir, "-lotprg", f"-Wl,-rpath,{libdir}", "-Wl,-rpath,/usr/local/cuda/lib64"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([str(exe)]).returncode == 0
