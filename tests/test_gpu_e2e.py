"""The end-to-end entry point fqnm_step_host (host buffer in, steps, host buffer out).
For one large periodic problem it runs the chunked pipeline (each chunk stepped on its
extended region [cC - H, cC + C + H) with H >= nsteps, copies overlapped with the
stepping on three streams): the result must equal the device-resident fqnm_step bit for
bit, the range check must still refuse out-of-range input, and small or non-periodic
plans take the plain path."""
import numpy as np
import pytest

import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    import paper_2604_06947_b200 as F
    return F


def _eo_plan(F, n, check=True):
    w = W.cfg("cfg4")
    q = W.q0_cfg4(n=1 << 31, count=n, device="cuda")
    qmax = int(q.abs().max())
    if check:
        plan = F.fqnm_plan(n, 1e-6, W.dt_dx_double(w, qmax), F.BURGERS_EO, F.PERIODIC)
    else:
        plan = F.fqnm_plan_ex(n, 1e-6, W.dt_dx_double(w, qmax), F.BURGERS_EO)
    return plan, q


@pytest.mark.parametrize("n,nsteps", [(1 << 24, 100), (1 << 24, 1), ((1 << 25) + (1 << 24), 257)])
@pytest.mark.parametrize("check", [True, False])
def test_pipelined_step_host_equals_device_path(F, n, nsteps, check):
    plan, q = _eo_plan(F, n, check)
    ref = q.clone()
    F.fqnm_step(plan, ref, nsteps)
    qh = torch.empty(n, dtype=torch.int32, pin_memory=True)
    qh.copy_(q.cpu())
    launches0 = plan.launches()
    F.fqnm_step_host(plan, qh, nsteps)
    assert plan.launches() > launches0
    assert torch.equal(qh, ref.cpu())
    # a second call reuses the pipeline (same nsteps) and continues the trajectory
    F.fqnm_step(plan, ref, nsteps)
    F.fqnm_step_host(plan, qh, nsteps)
    assert torch.equal(qh, ref.cpu())


def test_pipelined_step_host_range_check(F):
    n = 1 << 24
    plan, q = _eo_plan(F, n, True)
    hi = plan.info()["q_hi"]
    qh = torch.empty(n, dtype=torch.int32, pin_memory=True)
    qh.copy_(q.cpu())
    qh[n // 2 + 12345] = hi + 1
    with pytest.raises(F.FqnmError) as e:
        F.fqnm_step_host(plan, qh, 50)
    assert e.value.status == 3                              # FQNM_ERR_RANGE


def test_plain_step_host_paths(F):
    # small periodic, transmissive and batched plans take the plain (single copy) path
    rng = np.random.default_rng(4)
    for kw in (dict(n=70001, boundary=W.PERIODIC), dict(n=(1 << 24) + 4, boundary=W.TRANSMISSIVE)):
        n = kw["n"]
        q0 = W.smooth_random(rng, n, 100000, 20000).astype(np.int32)
        plan = F.fqnm_plan(n, 1e-5, 4 / 15, F.BURGERS_EO, kw["boundary"])
        ref = torch.tensor(q0, device="cuda")
        F.fqnm_step(plan, ref, 33)
        qh = torch.tensor(q0).pin_memory()
        F.fqnm_step_host(plan, qh, 33)
        assert torch.equal(qh, ref.cpu())


def _right_dependent_plans(F, n):
    """Plans whose update reads the right neighbour (the pipelined path's right
    halo must be exact, which strictly positive EO data never exercises)."""
    rng = np.random.default_rng(11)
    q_signed = W.smooth_random(rng, n, 100000, 0).astype(np.int32)      # changes sign
    qmax = int(np.abs(q_signed).max())
    lam_eo = W.dt_dx_double(W.cfg("cfg2"), qmax)
    yield "eo_signed", F.fqnm_plan(n, 1e-5, lam_eo, F.BURGERS_EO, F.PERIODIC), q_signed
    yield "lf", F.fqnm_plan_ex(n, 1e-3, 0.5, F.BURGERS_LF, flux_param=1.0,
                               q_range=(-900, 900)), np.clip(q_signed // 100, -900, 900)
    yield "linear_neg", F.fqnm_plan_ex(n, 1e-5, 0.5, F.LINEAR, flux_param=-1.0), q_signed
    yield "godunov", F.fqnm_plan_ex(n, 1e-5, lam_eo, F.BURGERS_GODUNOV), q_signed


@pytest.mark.parametrize("nsteps", [1, 37, 200])
def test_pipelined_step_host_right_neighbour_rules(F, nsteps):
    n = 1 << 24
    for name, plan, q0 in _right_dependent_plans(F, n):
        ref = torch.tensor(np.ascontiguousarray(q0, dtype=np.int32), device="cuda")
        l0 = plan.launches()
        F.fqnm_step(plan, ref, nsteps)
        dev_launches = plan.launches() - l0
        qh = torch.tensor(np.ascontiguousarray(q0, dtype=np.int32)).pin_memory()
        l0 = plan.launches()
        F.fqnm_step_host(plan, qh, nsteps)
        host_launches = plan.launches() - l0
        assert torch.equal(qh, ref.cpu()), name
        if name == "eo_signed":
            assert host_launches > 2 * dev_launches, "expected the chunked pipeline"
        # twice in a row (reused pipeline, continued trajectory)
        F.fqnm_step(plan, ref, nsteps)
        F.fqnm_step_host(plan, qh, nsteps)
        assert torch.equal(qh, ref.cpu()), name


def test_step_host_checks_buffer(F):
    plan = F.fqnm_plan(4096, 1e-5, 0.25, F.BURGERS_EO, F.PERIODIC)
    with pytest.raises(TypeError):
        F.fqnm_step_host(plan, torch.zeros(4096, dtype=torch.int64), 1)
    with pytest.raises(ValueError):
        F.fqnm_step_host(plan, torch.zeros(4095, dtype=torch.int32), 1)
    with pytest.raises(TypeError):
        F.fqnm_step_host(plan, np.zeros(4096, dtype=np.float32), 1)
    with pytest.raises(ValueError):
        F.fqnm_step_host(plan, np.zeros(8192, dtype=np.int32), 1)


@pytest.mark.parametrize("sign", [1, -1, 0])
def test_pipelined_step_host_sign_chunks(F, sign):
    """The pipelined fqnm_step_host on all-positive, all-negative and partly negative data
    (chunks of both kinds; the range-sign guard runs per chunk) equals fqnm_step, which
    itself runs K2S on the one-signed states."""
    n = 1 << 24
    rng = np.random.default_rng(5 + sign)
    q0 = np.abs(W.smooth_random(rng, n, 100000, 50000)).astype(np.int32)
    if sign < 0:
        q0 = -q0
    elif sign == 0:
        q0[: n // 3] = -q0[: n // 3]                      # some chunks mixed or negative
    qmax = int(np.abs(q0).max())
    lam = W.dt_dx_double(W.cfg("cfg2"), qmax)
    plan = F.fqnm_plan(n, 1e-5, lam, F.BURGERS_EO, F.PERIODIC)
    ref = torch.tensor(q0, device="cuda")
    F.fqnm_step(plan, ref, 77)
    qh = torch.tensor(q0).pin_memory()
    F.fqnm_step_host(plan, qh, 77)
    assert torch.equal(qh, ref.cpu())


@pytest.mark.parametrize("n,B", [(1024, 6000), (1000, 5003), (32, 40000)])
def test_step_host_ensemble_pipeline(F, n, B):
    """fqnm_step_host on an ensemble plan (warp kernel for n = 32 V, CTA kernel otherwise) runs
    the chunked copy / step / copy pipeline over whole problems; the result equals the
    device-resident fqnm_step, twice in a row on the same plan (the events are reused)."""
    rng = np.random.default_rng(n + B)
    q0 = rng.integers(-5000, 5000, size=(B, n)).astype(np.int32)
    plan = F.fqnm_plan_ex(n, 1e-4, 0.5, F.LINEAR, batch=B)
    assert plan.info()["kernel"] in (3, 4)
    ref = torch.tensor(q0, device="cuda")
    qh = torch.tensor(q0).pin_memory()
    for _ in range(2):
        F.fqnm_step(plan, ref, 53)
        F.fqnm_step_host(plan, qh, 53)
        assert torch.equal(qh, ref.cpu())
