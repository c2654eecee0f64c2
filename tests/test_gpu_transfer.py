"""GPU: the two transfer kernels (tensor-map TMA boxes, the default for n >= 10; per-element
loads, QAP_FLAG_LDG_TRANSFER) perform the same operations per class (reading R11): whole
dual states after bounds are bit-identical, for even and odd n (odd n - 2 shifts the TMA box
start to an even entry), at the root and at fixed nodes."""
import numpy as np
import pytest

import qapgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    import paper_1510_02065_b200 as p
    return p


@pytest.mark.parametrize("n,fixed", [(10, ()), (11, ()), (12, ((3, 1),)), (13, ()), (17, ((0, 16), (5, 2))),
                                     (24, ()), (30, ())])
def test_tma_transfer_equals_ldg(pkg, n, fixed):
    inst = qapgen.taib(n, 2) if n % 2 else qapgen.nug(n, 2)
    out = []
    for fl in (0, pkg.QAP_FLAG_LDG_TRANSFER):
        h = pkg.qap_rlt2_create(n, inst.F, inst.D, flags=fl)
        pkg.qap_rlt2_fix(h, list(fixed))
        r = pkg.qap_rlt2_bound(h, 3 if n < 24 else 2, trace=True)
        B, C, D, lb = pkg.qap_rlt2_dual_copy(h)
        out.append((r["trace"], B, C, D, lb))
        pkg.qap_destroy(h)
    (ta, Ba, Ca, Da, la), (tb, Bb, Cb, Db, lb_) = out
    assert la == lb_ and (ta == tb).all()
    assert (Ba == Bb).all() and (Ca == Cb).all() and np.array_equal(Da, Db)


def test_large_n_beyond_32bit_indices(pkg):
    """N = 48: 5.4e9 stored D entries (> 2^32) — element offsets are 64-bit per view base.
    Constant-cost instance: every permutation costs the same, so the GLB is that cost and
    every later LB' is 0 (closed form); both transfer kernels agree bit for bit."""
    import math
    n = 48
    c = qapgen.const(n, 2)
    opt = c.evaluate(list(range(n)))
    lbs = []
    for fl in (0, pkg.QAP_FLAG_LDG_TRANSFER):
        h = pkg.qap_rlt2_create(n, c.F, c.D, flags=fl)
        r = pkg.qap_rlt2_bound(h, 1, trace=True)
        assert r["lb_glb"] == opt and r["trace"][0] == opt
        lbs.append(r["lb"])
        pkg.qap_destroy(h)
    inst = qapgen.taib(n, 1)
    out = []
    for fl in (0, pkg.QAP_FLAG_LDG_TRANSFER):
        h = pkg.qap_rlt2_create(n, inst.F, inst.D, flags=fl)
        out.append(pkg.qap_rlt2_bound(h, 1)["lb"])
        B, C, _, _ = pkg.qap_rlt2_dual_copy(h, want_D=False)
        out.append((B.copy(), C.copy()))
        pkg.qap_destroy(h)
    assert out[0] == out[2] and math.isfinite(out[0])
    assert (out[1][0] == out[3][0]).all() and (out[1][1] == out[3][1]).all()


def test_capacity_refused(pkg):
    """N = 64 needs ~250 GB for D: refused with QAP_E_CAPACITY, no crash."""
    inst = qapgen.nug(64, 1)
    with pytest.raises(pkg.QapError) as ei:
        pkg.qap_rlt2_create(64, inst.F, inst.D)
    assert ei.value.status == 2  # QAP_E_CAPACITY
