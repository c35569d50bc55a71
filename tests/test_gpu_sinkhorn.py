"""GPU Sinkhorn baseline against the UNMODIFIED
reference sinkhorn (oracle/_ref, src/sinkhorn.cpp:69-151).

Floating-point parity: the device sums in a fixed parallel order and CUDA's
exp is not glibc's, so results agree to a tolerance, stated here: iteration
count within 1, relative 1e-9 on the plan cost, 1e-12 absolute on every plan
mass, identical plan sparsity; error classes and messages identical."""
import ctypes as C

import numpy as np
import pytest

from golden_util import random_instance

pytestmark = pytest.mark.gpu

otprg = pytest.importorskip("paper_2203_03732_b200")


def _ref(reference, mu, nu, cost, reg, max_iters=10000, tol=1e-9):
    L = reference.lib
    L.ref_sinkhorn.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                               C.c_int32, C.c_double] + [C.c_void_p] * 8 + [C.c_int64, C.c_void_p]
    n_a, n_b = cost.shape
    it, conv = C.c_int32(), C.c_int32()
    viol, pc, ms = C.c_double(), C.c_double(), C.c_double()
    ne = C.c_int64()
    cap = n_a * n_b
    ea, eb, em = np.empty(cap, np.int32), np.empty(cap, np.int32), np.empty(cap)
    st = L.ref_sinkhorn(n_a, n_b, mu.ctypes.data, nu.ctypes.data, cost.ctypes.data, reg, max_iters, tol,
                        C.byref(it), C.byref(conv), C.byref(viol), C.byref(pc), C.byref(ne),
                        ea.ctypes.data, eb.ctypes.data, em.ctypes.data, cap, C.byref(ms))
    if st:
        return st, L.ref_last_error().decode() if hasattr(L, "ref_last_error") else ""
    n = ne.value
    return 0, dict(iters=it.value, converged=bool(conv.value), violation=viol.value, cost=pc.value,
                   a=ea[:n], b=eb[:n], mass=em[:n], ms=ms.value)


def _instances():
    r = otprg.gen_random_ot_rational(60, 50, 3)
    yield "rational60x50", r.mu, r.nu, r.cost
    r = otprg.gen_random_ot_rational(120, 120, 7)
    yield "rational120", r.mu, r.nu, r.cost
    sq = otprg.gen_uniform_square(100, 2, dense=True)
    yield "square100", np.full(100, 0.01), np.full(100, 0.01), sq.cost


@pytest.mark.parametrize("reg", [0.05, 0.02])
def test_sinkhorn_matches_reference(reference, reg):
    for name, mu, nu, cost in _instances():
        st, ref = _ref(reference, mu, nu, cost, reg)
        assert st == 0, (name, ref)
        res = otprg.sinkhorn(otprg.OTInstance(mu, nu, cost), otprg.SinkhornConfig(reg=reg))
        assert abs(res.iters - ref["iters"]) <= 1, (name, res.iters, ref["iters"])
        assert res.converged == ref["converged"]
        assert res.cost == pytest.approx(ref["cost"], rel=1e-9), name
        assert np.array_equal(res.plan.a, ref["a"]) and np.array_equal(res.plan.b, ref["b"]), name
        assert np.max(np.abs(res.plan.mass - ref["mass"])) <= 1e-12, name
        # exact marginals after rounding (sinkhorn.cpp:12-66)
        assert np.allclose(res.plan.row_sums(len(mu)), mu, atol=1e-12)


def test_sinkhorn_iteration_cap_and_errors(reference):
    r = otprg.gen_random_ot_rational(40, 30, 5)
    inst = otprg.OTInstance(r.mu, r.nu, r.cost)
    res = otprg.sinkhorn(inst, otprg.SinkhornConfig(reg=0.01, max_iters=3))
    st, ref = _ref(reference, r.mu, r.nu, r.cost, 0.01, max_iters=3)
    assert res.iters == ref["iters"] == 3 and not res.converged and not ref["converged"]
    assert res.marginal_violation == pytest.approx(ref["violation"], rel=1e-6)
    with pytest.raises(otprg.ParameterError):
        otprg.sinkhorn(inst, otprg.SinkhornConfig(reg=0.0))
    with pytest.raises(otprg.ParameterError):
        otprg.sinkhorn(inst, otprg.SinkhornConfig(reg=0.1, tol=0.0))
    # regularisation so small the kernel underflows (sinkhorn.cpp:84-95)
    st, msg = _ref(reference, r.mu, r.nu, r.cost, 1e-4)
    assert st == 4
    with pytest.raises(otprg.NumericalError) as e:
        otprg.sinkhorn(inst, otprg.SinkhornConfig(reg=1e-4))
    assert str(e.value) == msg


def test_sinkhorn_scale_smoke():
    """n = 2,000 rational instance: converges with exact marginals."""
    r = otprg.gen_random_ot_rational(2000, 2000, 1)
    res = otprg.sinkhorn(otprg.OTInstance(r.mu, r.nu, r.cost),
                         otprg.SinkhornConfig(reg=otprg.reg_for_eps(0.05, 2000)), entries=False)
    assert res.converged and res.iters > 1 and res.device["n_entries"] > 0
