"""SURVEY §8(f) row f3 on the GPU: vks_mcmc_relocate / vks_mcmc_noise (through the C ABI) vs the
oracle (readings R1-R5 of DESIGN.md §4.7).

Relocation targets are integer decisions taken from exactly computed weights: bit-exact.  Copied
rows are exact copies; the split opacity logits are fp64 expressions rounded to fp32 on both sides
(CUDA and glibc pow / log may differ in the last fp64 ulp): within 1 fp32 ulp.  Noise: fp64 on
both sides from the same generator, rounded to fp32: within 2 ulp of the mean plus 1e-6 of the
displacement."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _scene(n, seed, dead_frac=0.2):
    s = synth.make_scene(n, "indoor", seed)
    rng = np.random.default_rng(seed)
    s["opacity_logits"][rng.random(n) < dead_frac] = -8.0
    return s


@pytest.mark.parametrize("n,seed", [(1, 0), (1000, 1), (123457, 2), (1000000, 3)])
def test_relocate_matches_oracle(n, seed):
    import torch
    import paper_2605_00219_b200 as P
    s = _scene(n, seed)
    K = s["sh"].shape[1]
    prm = P.GaussianParams.from_host(s)
    groups = [prm.means, prm.log_scales, prm.quats, prm.opacity_logits, prm.sh]
    m = [torch.rand_like(t) for t in groups]
    v = [torch.rand_like(t) for t in groups]
    m_host = np.concatenate([t.cpu().numpy().reshape(-1) for t in m])
    tg = torch.empty(n, dtype=torch.int64, device="cuda")
    nd = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(P.vks_mcmc_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    P.vks_mcmc_relocate(prm, ws, dead_opacity=0.005, seed=seed + 17, m=m, v=v, targets=tg, n_dead=nd)
    torch.cuda.synchronize()
    out, tgo, ndo, mo, _ = oracle.mcmc_relocate(s, 0.005, seed + 17, m=m_host, v=m_host.copy())
    assert int(nd.item()) == ndo
    assert np.array_equal(tg.cpu().numpy(), tgo)
    for k, t in zip(("means", "log_scales", "quats", "sh"), (prm.means, prm.log_scales, prm.quats, prm.sh)):
        assert np.array_equal(t.cpu().numpy(), out[k]), k
    lg, lo = prm.opacity_logits.cpu().numpy(), out["opacity_logits"]
    ulp = np.spacing(np.abs(lo).astype(np.float32))
    assert np.all(np.abs(lg.astype(np.float64) - lo) <= ulp), int((np.abs(lg - lo) > ulp).sum())
    mg = np.concatenate([t.cpu().numpy().reshape(-1) for t in m])
    assert np.array_equal(mg, mo)


def test_noise_matches_oracle():
    import torch
    import paper_2605_00219_b200 as P
    n = 200003
    s = _scene(n, 9, dead_frac=0.5)
    prm = P.GaussianParams.from_host(s)
    P.vks_mcmc_noise(prm, 1.6e-4, 5e5, seed=21, step=7)
    torch.cuda.synchronize()
    ref = oracle.mcmc_noise(s, 1.6e-4, 5e5, seed=21, step=7).astype(np.float64)
    got = prm.means.cpu().numpy().astype(np.float64)
    disp = np.abs(ref - s["means"].astype(np.float64))
    tol = 2 * np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64) + 1e-6 * disp
    assert np.all(np.abs(got - ref) <= tol), int((np.abs(got - ref) > tol).sum())
    assert (disp > 0).sum() > n // 4  # the dead half moved


def test_relocate_degenerate_budgets():
    """Every Gaussian dead (no alive weight): nothing moves and every target is -1; nobody dead:
    the parameters are untouched."""
    import torch
    import paper_2605_00219_b200 as P
    for logit in (-9.0, 3.0):
        s = _scene(4097, 5, dead_frac=0.0)
        s["opacity_logits"][:] = logit
        prm = P.GaussianParams.from_host(s)
        before = [t.clone() for t in (prm.means, prm.log_scales, prm.quats, prm.opacity_logits, prm.sh)]
        tg = torch.empty(4097, dtype=torch.int64, device="cuda")
        nd = torch.zeros(1, dtype=torch.int64, device="cuda")
        ws = torch.empty(P.vks_mcmc_workspace_bytes(4097), dtype=torch.uint8, device="cuda")
        P.vks_mcmc_relocate(prm, ws, dead_opacity=0.005, seed=1, targets=tg, n_dead=nd)
        torch.cuda.synchronize()
        assert int(nd.item()) == (4097 if logit < 0 else 0)
        assert bool((tg == -1).all())
        for a, b in zip(before, (prm.means, prm.log_scales, prm.quats, prm.opacity_logits, prm.sh)):
            assert torch.equal(a, b)
