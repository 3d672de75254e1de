"""Host-resident dense source (cabs.h: cabs_source.host_resident = 1): A stays in pinned host
memory, the library reads only what Algorithm 2 samples ("never knowing the remaining
entries") through the mapped address.  Everything must equal the device-resident run bit
for bit (the gathers are exact copies); the sampled residual too (same pairs, same entries); the
exact residual (plain loads over the interconnect) matches the FP64 oracle within the parity
tolerance.  Pin P12's idea on the GPU: entries outside the sampled rows / columns are poisoned
with NaN in the host copy and the sketch must not change."""
import ctypes
import math

import numpy as np
import pytest
import torch

from oracle import cabs as O

pytestmark = pytest.mark.gpu

C = pytest.importorskip("paper_1607_07395_b200.cabs")

EXACT_KEYS = ("I", "J", "C", "R", "W", "s1", "P", "Q", "cen_r", "cen_c", "lab_r", "lab_c", "Ib", "Jb", "U", "V", "s2")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    C.load()
    return torch.device("cuda:0")


def _A(m, n, seed):
    g = np.random.default_rng(seed)
    r = 24
    A = (g.standard_normal((m, r)) / np.arange(1, r + 1)) @ g.standard_normal((r, n)) + 0.01 * g.standard_normal((m, n))
    return A.astype(np.float32)


@pytest.mark.parametrize("m,n,k1,k2,iters,samples", [(3001, 2003, 40, 50, 6, 0), (2048, 1024, 100, 100, 4, 100000),
                                                     (700, 1900, 16, 24, 5, 0)])
def test_host_resident_pipeline_identical_to_device(dev, m, n, k1, k2, iters, samples):
    from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline
    A = _A(m, n, 3 * m + n)
    cfg = CabsConfig(k1, k2, iters, seed=6, residual_samples=samples)
    a = CabsPipeline(torch.from_numpy(A).to(dev), m, n, cfg)
    a.run()
    ga = a.results()
    b = CabsPipeline(C.HostDense(torch.from_numpy(A).pin_memory(), dev), m, n, cfg)
    b.run()
    gb = b.results()
    for key in EXACT_KEYS:
        assert torch.equal(ga[key], gb[key]), key
    if samples:
        assert torch.equal(a.out, b.out)
    else:
        r2 = gb["r2"]
        r_or, a_or = O.residual(A, gb["U"].numpy()[:, :r2], gb["V"].numpy()[:, :r2], gb["s2"].numpy()[:r2])
        assert abs(gb["a_sq"] - a_or) <= 1e-6 * a_or
        assert abs(math.sqrt(gb["resid_sq"]) - math.sqrt(r_or)) <= 1e-4 * math.sqrt(r_or) + 1e-6 * math.sqrt(a_or)


@pytest.mark.parametrize("host", [False, True])
@pytest.mark.parametrize("m,n,k1,k2,iters,pad", [(3001, 2003, 40, 50, 6, 0), (1500, 2600, 100, 100, 4, 3)])
def test_dual_layout_identical_to_single(dev, host, m, n, k1, k2, iters, pad):
    # cabs_source.at: the column gathers read the column-major copy (device or pinned host memory)
    from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline
    A = _A(m, n, m + 5 * n)
    cfg = CabsConfig(k1, k2, iters, seed=8)
    A_d = torch.from_numpy(A).to(dev)
    a = CabsPipeline(A_d, m, n, cfg)
    a.run()
    ga = a.results()
    At = torch.full((n, m + pad), float("nan"))
    At[:, :m] = torch.from_numpy(A).t()
    if host:
        src = C.HostDense(torch.from_numpy(A).pin_memory(), dev, At=At.pin_memory()[:, :m])
    else:
        src = C.DualDense(A_d, At.to(dev)[:, :m])
    b = CabsPipeline(src, m, n, cfg)
    b.run()
    gb = b.results()
    for key in EXACT_KEYS:
        assert torch.equal(ga[key], gb[key]), key
    assert C.cabs_device_status(b.ws) == 0
    if not host:  # the exact residual reads `a` only: the same kernel on the same bytes
        assert gb["resid_sq"] == ga["resid_sq"] and gb["a_sq"] == ga["a_sq"]


def test_dual_layout_column_gather_reads_the_second_copy(dev):
    # C must come from `at`, R from `a`: make the two copies differ on purpose and look at C and R
    m, n, k = 600, 400, 12
    from paper_1607_07395_b200.dist import make_plan
    plan = make_plan(m, n, k, 0, 1)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    A = torch.from_numpy(_A(m, n, 1)).to(dev)
    At = (A + 1.0).t().contiguous()
    I = torch.zeros(k, dtype=torch.int64, device=dev)
    J = torch.zeros(k, dtype=torch.int64, device=dev)
    ld = C.cabs_padded_ld(k)
    Cm, R, W = torch.zeros((m, ld), device=dev), torch.zeros((k, n), device=dev), torch.zeros((k, ld), device=dev)
    C.cabs_pilot(plan, C.DualDense(A, At), k, 2, I, J, Cm, R, W, ws)
    assert torch.equal(Cm[:, :k], (A + 1.0)[:, J])
    assert torch.equal(R, A[I, :])


def test_host_resident_sketch_reads_only_sampled_entries(dev):
    # linear access: poison every entry outside the rows / columns the run sampled
    from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline
    m, n = 2500, 1700
    A = _A(m, n, 5)
    cfg = CabsConfig(30, 30, 5, seed=9)
    a = CabsPipeline(C.HostDense(torch.from_numpy(A).pin_memory(), dev), m, n, cfg)
    a.run(with_residual=False)
    ga = a.results()
    rows = np.union1d(ga["I"].numpy(), ga["Ib"].numpy())
    cols = np.union1d(ga["J"].numpy(), ga["Jb"].numpy())
    Ap = np.full_like(A, np.nan)
    Ap[rows, :] = A[rows, :]
    Ap[:, cols] = A[:, cols]
    b = CabsPipeline(C.HostDense(torch.from_numpy(Ap).pin_memory(), dev), m, n, cfg)
    b.run(with_residual=False)
    gb = b.results()
    for key in EXACT_KEYS:
        assert torch.equal(ga[key], gb[key]), key
    assert C.cabs_device_status(b.ws) == 0  # no non-finite value was ever read


def test_host_resident_argument_errors(dev):
    m, n, k = 200, 100, 10
    from paper_1607_07395_b200.dist import make_plan
    plan = make_plan(m, n, k, 0, 1)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    I = torch.zeros(k, dtype=torch.int64, device=dev)
    J = torch.zeros(k, dtype=torch.int64, device=dev)
    ld = C.cabs_padded_ld(k)
    Cm, R, W = torch.zeros((m, ld), device=dev), torch.zeros((k, n), device=dev), torch.zeros((k, ld), device=dev)
    L = C.load()
    host = torch.zeros((m, n)).pin_memory()

    def pilot(src):
        return L.cabs_pilot(ctypes.byref(plan), ctypes.byref(src), k, 0, I.data_ptr(), J.data_ptr(), Cm.data_ptr(), ld,
                            R.data_ptr(), n, W.data_ptr(), ld, ws.data_ptr(), ws.numel(), None, None)

    assert pilot(C._source(C.HostDense(host, dev))) == 0
    bad = C._source(C.HostDense(host, dev)); bad.host_resident = 3
    assert pilot(bad) == 1  # CABS_ERR_INVALID_ARG
    x, y = torch.zeros((m, 3), device=dev), torch.zeros((n, 3), device=dev)
    rbf = C._source(C.RbfSource(x, y, 1.0)); rbf.host_resident = 1
    assert pilot(rbf) == 1
    dual = C._source(C.HostDense(host, dev, At=torch.zeros((n, m)).pin_memory())); dual.ldat = m - 1
    assert pilot(dual) == 1
    dual = C._source(C.HostDense(host, dev, At=torch.zeros((n, m)).pin_memory())); dual.transposed = 1
    assert pilot(dual) == 1
    torch.cuda.synchronize()
    with pytest.raises(TypeError):
        C.HostDense(torch.zeros((4, 4)), dev)  # not pinned
