"""Engine edge cases found in review: graph runs after an odd
number of host steps, same-shape data swaps that change a captured kernel
argument, several handles with different fused-resampling shared memory, and
the resampler's per-call destination buffers."""
import numpy as np
import pytest

import inputs
import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["crbd_lr", "clads2_lr", "seir"])
@pytest.mark.parametrize("n_steps", [1, 3])
def test_run_after_odd_steps_matches_oracle(smc, kind, n_steps):
    t90 = inputs.tree("tree90")
    N, seed = 2000, 5
    if kind == "crbd_lr":
        m, ok, data, prm = smc.Model.crbd(t90, lineage=True), oracle.CRBD_LR, oracle.tree_blob(t90), inputs.CRBD_PARAMS
    elif kind == "clads2_lr":
        m, ok, data, prm = smc.Model.clads2(t90, lineage=True), oracle.CLADS2_LR, oracle.tree_blob(t90), inputs.CLADS2_PARAMS
    else:
        y = inputs.seir_series()
        m, ok, data, prm = smc.Model.seir(y), oracle.SEIR, y, None
    g = smc.Smc(m, N, seed)
    for _ in range(n_steps):
        rc, done = g.step()
        assert rc == smc.OK and not done
    assert g.run_status() == smc.OK          # graph path from an odd parity
    o = oracle.Smc(ok, data, prm, N, seed)
    assert o.run() == oracle.OK
    assert g.log_z == pytest.approx(o.log_z, rel=1e-9)
    np.testing.assert_array_equal(g.ancestors(), o.anc())


def _mirror_root(tree):
    t = {k: (list(v) if isinstance(v, list) else v) for k, v in tree.items()}
    r = t["root"]
    t["left"][r], t["right"][r] = t["right"][r], t["left"][r]
    return t


def test_set_data_new_root_order_recaptures_graph(smc):
    t90 = inputs.tree("tree90")
    mir = _mirror_root(t90)
    N, seed = 2000, 9
    g = smc.Smc(smc.Model.clads2(t90, lineage=True), N, seed)
    assert g.run_status() == smc.OK          # graph captured with the original root order
    g.set_data(smc.tree_data(mir))
    g.reset(seed)
    assert g.run_status() == smc.OK
    ref = smc.Smc(smc.Model.clads2(mir, lineage=True), N, seed)
    assert ref.run_status() == smc.OK
    assert g.log_z == ref.log_z
    np.testing.assert_array_equal(g.fields(), ref.fields())


def test_fused_handles_of_different_sizes(smc):
    t90 = inputs.tree("tree90")
    big = smc.Smc(smc.Model.crbd(t90, lineage=True), 2_000_000, 3)
    small = smc.Smc(smc.Model.crbd(t90, lineage=True), 1000, 3)
    assert big.resample_grid() > 0 and small.resample_grid() > 0
    assert small.run_status() == smc.OK
    assert big.run_status() == smc.OK          # its launches still get their shared memory


def test_resample_device_does_not_redirect_handle(smc):
    import torch
    n, S = 5000, 64
    lw = inputs.resample_lw(n, 1.0, 0.1, seed=4)
    st = inputs.state_bytes(n, S, seed=5)
    r = smc.Resampler(n, S, seed=4)
    d_lw = torch.tensor(lw, device="cuda")
    d_in = torch.tensor(smc.aos_to_soa(st), device="cuda")
    d_out = torch.empty_like(d_in)
    d_anc = torch.empty(n, dtype=torch.int32, device="cuda")
    r.device(d_lw, d_in, d_out, d_anc, epoch=0, sync_logz=True)
    del d_out, d_anc                          # the caller's buffers go away
    torch.cuda.synchronize()
    anc, out, _ = r.host(lw, smc.aos_to_soa(st), epoch=0)
    ref = oracle.resample(lw, seed=4, epoch=0)["anc"]
    np.testing.assert_array_equal(anc, ref)
    np.testing.assert_array_equal(smc.soa_to_aos(out), st[ref])
    with pytest.raises(smc.SmcError):
        r.device(d_lw.data_ptr() + 8, d_in, d_in, torch.empty(n, dtype=torch.int32, device="cuda"))
