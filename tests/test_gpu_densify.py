"""SURVEY §8(f) row f4 on the GPU: vks_densify_stats / vks_densify (through the C ABI) vs the
oracle (readings R6-R9 of DESIGN.md §4.7).  Decisions (prune / keep / clone /
split) and the row order are exact; copied rows and moments bit-exact; split children's fp64
positions and log-scales rounded to fp32 on both sides (CUDA vs glibc transcendentals may differ
in the last fp64 ulp): within 1 fp32 ulp; the statistics within 1 fp32 ulp per view."""
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


def _ulp_close(a, b, ulps=1):
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    return np.all(np.abs(a64 - b64) <= ulps * np.spacing(np.abs(b).astype(np.float32)).astype(np.float64))


@pytest.mark.parametrize("n,seed", [(1, 0), (5000, 1), (300001, 2)])
def test_densify_matches_oracle(n, seed):
    import torch
    import paper_2605_00219_b200 as P
    s = synth.make_scene(n, "outdoor", seed)
    rng = np.random.default_rng(seed)
    s["opacity_logits"][rng.random(n) < 0.1] = -7.0  # prunable
    K = s["sh"].shape[1]
    G = oracle.ADAM_GROUPS
    prm = [torch.from_numpy(np.ascontiguousarray(s[k])).cuda() for k in G]
    m = [torch.rand_like(t) for t in prm]
    v = [torch.rand_like(t) for t in prm]
    # statistics from two "views" of random 2D gradients, half the Gaussians visible in each
    accum = torch.zeros(n, device="cuda")
    denom = torch.zeros(n, device="cuda")
    a_h, d_h = np.zeros(n, np.float32), np.zeros(n, np.float32)
    for view in range(2):
        g2 = (rng.normal(size=(n, 2)) * 3e-4).astype(np.float32)
        rad = np.where(rng.random((n, 1)) < 0.5, 4, 0).repeat(2, 1).astype(np.int32)
        P.vks_densify_stats(torch.from_numpy(g2).cuda(), torch.from_numpy(rad).cuda(), accum, denom)
        a_h, d_h = oracle.densify_stats(g2, rad, a_h, d_h)
    torch.cuda.synchronize()
    assert _ulp_close(accum.cpu().numpy(), a_h) and np.array_equal(denom.cpu().numpy(), d_h)
    gthr, sthr = 2e-4, float(np.median(np.exp(s["log_scales"]).max(1)))  # half clone, half split
    cap = 2 * n
    out = [torch.empty((cap,) + tuple(t.shape[1:]), device="cuda") for t in prm]
    om = [torch.empty_like(t) for t in out]
    ov = [torch.empty_like(t) for t in out]
    ws = torch.empty(P.vks_densify_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    n2 = P.vks_densify(prm, accum, denom, out, ws, gthr, sthr, 0.005, seed=seed + 1, m=m, v=v, out_m=om, out_v=ov)
    torch.cuda.synchronize()
    m_host = np.concatenate([t.cpu().numpy().reshape(-1) for t in m])
    ref, n2o, mo, vo = oracle.densify(s, a_h, d_h, gthr, sthr, 0.005, seed=seed + 1, m=m_host,
                                      v=np.concatenate([t.cpu().numpy().reshape(-1) for t in v]))
    assert n2 == n2o
    for k, t in zip(G, out):
        got = t[:n2].cpu().numpy()
        if k in ("means", "log_scales"):
            assert _ulp_close(got, ref[k]), k
        else:
            assert np.array_equal(got, ref[k]), k
    mg = np.concatenate([t[:n2].cpu().numpy().reshape(-1) for t in om])
    vg = np.concatenate([t[:n2].cpu().numpy().reshape(-1) for t in ov])
    assert np.array_equal(mg, mo) and np.array_equal(vg, vo)


def test_densify_capacity_protocol():
    """R9: n' above the output capacity -> VKS_ERR_CAPACITY with n' reported, nothing written; a
    call with grown outputs (x1.5) succeeds with the same n'."""
    import torch
    import paper_2605_00219_b200 as P
    n = 1000
    s = synth.make_scene(n, "outdoor", 5)
    s["opacity_logits"] = np.maximum(s["opacity_logits"], -3.0).astype(np.float32)
    prm = [torch.from_numpy(np.ascontiguousarray(s[k])).cuda() for k in oracle.ADAM_GROUPS]
    accum, denom = torch.ones(n, device="cuda"), torch.ones(n, device="cuda")
    ws = torch.empty(P.vks_densify_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    small = [torch.full((n + 10,) + tuple(t.shape[1:]), 7.0, device="cuda") for t in prm]
    with pytest.raises(P.VksError) as ei:
        P.vks_densify(prm, accum, denom, small, ws, 0.5, 1e9)  # everything clones: n' = 2n
    assert ei.value.status == 2 and ei.value.n_out == 2 * n
    assert all(bool((t == 7.0).all()) for t in small)
    cap = int(1.5 * (n + 10)) + n
    big = [torch.empty((cap,) + tuple(t.shape[1:]), device="cuda") for t in prm]
    assert P.vks_densify(prm, accum, denom, big, ws, 0.5, 1e9) == 2 * n


def test_densify_prunes_everything_and_keeps_everything():
    """Every Gaussian below the prune opacity -> n' = 0; none above the gradient threshold and none
    prunable -> the rows come back unchanged."""
    import torch
    import paper_2605_00219_b200 as P
    n = 3001
    s = synth.make_scene(n, "outdoor", 6)
    G = oracle.ADAM_GROUPS
    ws = torch.empty(P.vks_densify_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    out = None
    for logit, expect in ((-8.0, 0), (2.0, n)):
        s["opacity_logits"][:] = logit
        prm = [torch.from_numpy(np.ascontiguousarray(s[k])).cuda() for k in G]
        out = [torch.empty((2 * n,) + tuple(t.shape[1:]), device="cuda") for t in prm]
        acc, den = torch.zeros(n, device="cuda"), torch.ones(n, device="cuda")
        assert P.vks_densify(prm, acc, den, out, ws, 1e-3, 0.01) == expect
        if expect:
            for a, b in zip(prm, out):
                assert torch.equal(a, b[:n])
