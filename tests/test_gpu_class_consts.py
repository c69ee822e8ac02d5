"""The class-size constants of every search kernel (tsa_class_consts): n^-q,
ln n and 1/n from the 33 KB table + Horner polynomial, checked
against the definition evaluated in 64-bit-mantissa long double on the host.

A class of n voxels contributes A = W / n^q (PAPER.md:581-591 with
p_i/P_j = c_i/n, R11) or S = ln n - W/n at q == 1 (R6).  The search
only needs these to be accurate (the reported objective is recomputed from the
definition by the finalize step), so the bar is 8 ulp (6 for 1/n), not bit equality;
n <= 2^11 reads the table entry itself and must equal 1/pow(n, q) as the
library's table computes it to within 1 ulp.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

QS = [0.05, 0.5, 0.8, 0.9999, 1.0, 1.2, 1.5, 2.5, 7.0, 12.0, 40.0]


def _ns():
    rng = np.random.default_rng(20121068)
    n = [np.arange(1, 8193, dtype=np.int64)]
    p = 2 ** np.arange(0, 31, dtype=np.int64)
    n += [p, p - 1, p + 1, p[:-1] * 3 // 2]
    n += [rng.integers(1, 2 ** 20 + 1, 200_000), rng.integers(1, 2 ** 31 - 1, 50_000)]
    n = np.concatenate(n)
    return np.unique(n[(n >= 1) & (n < 2 ** 31)])


def _ulp_err(got, ref):
    ref64 = ref.astype(np.float64)
    return np.abs(got.astype(np.longdouble) - ref) / np.spacing(np.abs(ref64)).astype(np.longdouble)


@pytest.mark.parametrize("q", QS)
def test_class_consts_vs_long_double(q):
    import paper_2012_10684_b200 as tsa

    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    n = _ns()
    dn = torch.from_numpy(n.astype(np.int32)).cuda()
    nl = n.astype(np.longdouble)
    if q != 1.0:
        a = tsa.tsa_class_consts(dn, q).cpu().numpy()
        ref = np.power(nl, -np.longdouble(q))
        ok = ref > np.longdouble(np.finfo(np.float64).tiny)  # normal range only
        err = _ulp_err(a[ok], ref[ok])
        assert float(err.max()) <= 8.0, (q, float(err.max()), n[ok][int(np.argmax(err))])
    else:
        a, b = tsa.tsa_class_consts(dn, q)
        a, b = a.cpu().numpy(), b.cpu().numpy()
        ref_ln = np.log(nl)
        big = n > 1  # ln 1 = 0 exactly
        assert np.all(a[~big] == 0.0)
        err = _ulp_err(a[big], ref_ln[big])
        assert float(err.max()) <= 8.0, float(err.max())
        err = _ulp_err(b, 1 / nl)
        assert float(err.max()) <= 6.0, float(err.max())


def test_class_consts_zero_is_nan():
    import paper_2012_10684_b200 as tsa

    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    dn = torch.tensor([0, 1, 2], dtype=torch.int32, device="cuda")
    a = tsa.tsa_class_consts(dn, 0.8).cpu().numpy()
    assert np.isnan(a[0]) and a[1] == 1.0
    a, b = tsa.tsa_class_consts(dn, 1.0)
    assert np.isnan(a[0].item()) and np.isnan(b[0].item()) and b[1].item() == 1.0
