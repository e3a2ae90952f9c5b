"""GPU parity of in-place resampling (R-21) against the
oracle's ancestor permutation, element by element: permuted ancestors
bit-exact, states bit-exact, log Z / log-weights to 1e-9."""
import math

import numpy as np
import pytest

import inputs
import oracle
from tests.test_gpu_parity import GPU_KIND, TREE_KINDS, compare, RTOL

pytestmark = pytest.mark.gpu


# ------------------------------------------------------------- resampler alone
@pytest.mark.parametrize("N", [1, 2, 7, 2047, 2048, 2049, 100_003])
@pytest.mark.parametrize("sigma,finf", [(0.0, 0.0), (1.0, 0.0), (4.0, 0.25), (12.0, 0.5)])
def test_inplace_resampler_parity(smc, N, sigma, finf):
    lw = inputs.resample_lw(N, sigma, finf, seed=N)
    if not np.isfinite(lw).any():
        lw[0] = 0.0
    S = 64
    st = inputs.state_bytes(N, S, seed=N + 1)
    r = smc.Resampler(N, S, seed=77, inplace=True)
    for epoch in (0, 5):
        anc, out, inc = r.host(lw, smc.aos_to_soa(st), epoch=epoch)
        ref = oracle.resample(lw, seed=77, epoch=epoch)
        c = oracle.permute(ref["anc"])
        np.testing.assert_array_equal(anc, c)
        assert inc == pytest.approx(ref["logz_inc"], rel=1e-13, abs=1e-13)
        np.testing.assert_array_equal(smc.soa_to_aos(out), oracle.gather(st, c))
        assert r.distinct() == len(np.unique(ref["anc"]))


@pytest.mark.parametrize("S", [16, 32, 96, 128, 272])
def test_inplace_state_sizes(smc, S):
    N = 5000
    lw = inputs.resample_lw(N, 2.0, 0.1, seed=3)
    st = inputs.state_bytes(N, S, seed=4)
    r = smc.Resampler(N, S, seed=5, inplace=True)
    anc, out, _ = r.host(lw, smc.aos_to_soa(st), epoch=2)
    c = oracle.permute(oracle.resample(lw, seed=5, epoch=2)["anc"])
    np.testing.assert_array_equal(anc, c)
    np.testing.assert_array_equal(smc.soa_to_aos(out), oracle.gather(st, c))


def test_inplace_device_buffers(smc):
    import torch
    N, S = (1 << 20) + 333, 64
    lw = inputs.resample_lw(N, 1.0, 0.0, seed=8)
    st = inputs.state_bytes(N, S, seed=9)
    dev = torch.device("cuda")
    d_lw = torch.from_numpy(lw).to(dev)
    d_st = torch.from_numpy(np.ascontiguousarray(smc.aos_to_soa(st))).to(dev)
    d_anc = torch.empty(N, dtype=torch.int32, device=dev)
    r = smc.Resampler(N, S, seed=6, stream=torch.cuda.current_stream(), inplace=True)
    inc = r.device(d_lw, d_st, None, d_anc, epoch=3, sync_logz=True)
    ref = oracle.resample(lw, seed=6, epoch=3)
    c = oracle.permute(ref["anc"])
    np.testing.assert_array_equal(d_anc.cpu().numpy().view(np.uint32), c)
    np.testing.assert_array_equal(smc.soa_to_aos(d_st.cpu().numpy()), oracle.gather(st, c))
    assert inc == pytest.approx(ref["logz_inc"], rel=1e-13)
    other = torch.empty_like(d_st)
    with pytest.raises(smc.SmcError) as e:
        r.device(d_lw, d_st, other, d_anc)
    assert e.value.code == smc.EINVAL


def test_inplace_single_heavy_particle(smc):
    N = 300_000
    lw = np.full(N, -np.inf)
    lw[123_457] = 0.0
    st = inputs.state_bytes(N, 64, seed=9)
    r = smc.Resampler(N, 64, seed=2, inplace=True)
    anc, out, _ = r.host(lw, smc.aos_to_soa(st))
    assert np.all(anc == 123_457)
    np.testing.assert_array_equal(smc.soa_to_aos(out), np.broadcast_to(st[123_457], st.shape))


# ------------------------------------------------------------- whole SMC runs
def both_inplace(smc, kind, data, params, N, seed):
    if kind in TREE_KINDS:
        gk, fl = GPU_KIND.get(kind, (kind, None))
        flags = (getattr(smc, fl) if fl else 0) | smc.FLAG_INPLACE
        gm = smc.Model(gk, smc.tree_data(data), params, flags=flags)
        od = oracle.tree_blob(data)
    else:
        gm = smc.Model(kind, data, params, flags=smc.FLAG_INPLACE)
        od = data
    o = oracle.Smc(kind, od, params, N, seed)
    o.set_inplace(True)
    return smc.Smc(gm, N, seed), o


def run_pair_inplace(smc, kind, data, params, N, seed, ess=None, per_epoch=True, max_epochs=None):
    g, o = both_inplace(smc, kind, data, params, N, seed)
    if ess:
        g.set_ess_threshold(*ess)
        o.set_ess(*ess)
    e = 0
    while True:
        rg, dg = g.step()
        ro, do = o.step()
        assert rg == ro and dg == do
        if per_epoch or dg:
            compare(g, o)
        e += 1
        if dg or (max_epochs and e >= max_epochs):
            break
    if dg and math.isfinite(o.log_z):
        assert g.log_z == pytest.approx(o.log_z, rel=RTOL)
        assert g.stats()["resamples"] == o.stats()["resamples"]
    return g, o


@pytest.mark.parametrize("kind,data,params,N,ess", [
    (oracle.CRBD, "tree5", inputs.CRBD_PARAMS, 1000, None),
    (oracle.CRBD, "tree5", inputs.CRBD_PARAMS, 2049, (1, 2)),
    (oracle.CRBD_LR, "tree90", inputs.CRBD_PARAMS, 3000, None),
    (oracle.CRBD_AE, "tree90", inputs.CRBD_PARAMS, 3000, (1, 2)),
    (oracle.CLADS2, "tree5", inputs.CLADS2_PARAMS, 2000, None),
    (oracle.SEIR, "seir", None, 1000, None),
    (oracle.GEOMETRIC, None, inputs.GEOMETRIC_PARAMS, 3001, None),
    (oracle.SSM, "ssm", inputs.SSM_PARAMS, 2000, (3, 4)),
    (oracle.CONSTW, None, inputs.CONSTW_PARAMS, 10, None),
    (oracle.FIG3, None, inputs.FIG3_PARAMS, 4001, None),
    (oracle.STACKF, "stackf", inputs.STACKF_PARAMS, 4001, None),
    (oracle.STACKF, "stackf", inputs.STACKF_PARAMS, 4001, (1, 2)),
])
def test_inplace_smc_parity(smc, kind, data, params, N, ess):
    data = {"tree5": lambda: inputs.tree("tree5"), "tree90": lambda: inputs.tree("tree90"),
            "seir": inputs.seir_series, "ssm": lambda: inputs.ssm_series(10),
            "stackf": inputs.stackf_series}.get(data, lambda: data)()
    run_pair_inplace(smc, kind, data, params, N, 11, ess=ess, per_epoch=kind != oracle.SEIR)


def test_inplace_full_size_prefix(smc):
    run_pair_inplace(smc, oracle.CRBD_LR, inputs.tree("tree90"), inputs.CRBD_PARAMS, 1_000_000, 1,
                     max_epochs=4)


def test_inplace_graph_run(smc):
    g, o = both_inplace(smc, oracle.CRBD_AE, inputs.tree("tree90"), inputs.CRBD_PARAMS, 5000, 3)
    g.set_ess_threshold(1, 2)
    o.set_ess(1, 2)
    g.set_graph(True)
    assert g.run_status() == smc.OK
    assert o.run() == oracle.OK
    compare(g, o)
    assert g.log_z == pytest.approx(o.log_z, rel=RTOL)


def test_inplace_needs_single_shard(smc):
    with pytest.raises(smc.SmcError) as e:
        smc.Smc(smc.Model.crbd(inputs.tree("tree5"), flags=smc.FLAG_INPLACE), 1000, 1, shards=2)
    assert e.value.code == smc.EINVAL
