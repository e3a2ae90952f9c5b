"""The real one-process-per-shard path on ONE GPU: two processes, host
all-gather over gloo for the records, CUDA IPC peer stores for migration.
Must be bit-identical to one process holding all particles (reading R1)."""
import numpy as np
import pytest

import inputs
from tests import dist_workers

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("lineage", [False, True])
def test_two_processes_one_gpu_match_single(smc, tmp_path, lineage):
    import torch.multiprocessing as mp
    n_per, seed = 3000, 17
    port = dist_workers.free_port()
    mp.spawn(dist_workers.gpu_worker, args=(2, port, str(tmp_path), n_per, seed, lineage), nprocs=2,
             join=True)
    g = [np.load(tmp_path / f"g{r}.npy", allow_pickle=True) for r in range(2)]
    ref = smc.Smc(smc.Model.crbd(inputs.tree("tree90"), lineage=lineage), 2 * n_per, seed)
    assert ref.run_status() == g[0][0] == g[1][0] == smc.OK
    assert g[0][1] == g[1][1] == ref.log_z
    np.testing.assert_array_equal(np.concatenate([g[0][2], g[1][2]]), ref.ancestors())
    np.testing.assert_array_equal(np.concatenate([g[0][3], g[1][3]]), ref.log_weights())
    np.testing.assert_array_equal(np.concatenate([g[0][4], g[1][4]]), ref.fields())
    assert g[0][5]["world"] == 2 and g[0][5]["rank"] == 0 and g[1][5]["rank"] == 1


def test_resample_two_processes_one_gpu(smc, tmp_path):
    import torch.multiprocessing as mp
    import oracle
    n_per = 4001
    port = dist_workers.free_port()
    mp.spawn(dist_workers.gpu_resample_worker, args=(2, port, str(tmp_path), n_per), nprocs=2,
             join=True)
    r = [np.load(tmp_path / f"rs{k}.npy", allow_pickle=True) for k in range(2)]
    N = 2 * n_per
    lw = inputs.resample_lw(N, 2.0, 0.2, seed=41)
    st = inputs.state_bytes(N, 64, seed=42)
    a0 = oracle.resample(lw, seed=7, epoch=0)["anc"]
    a1 = oracle.resample(lw, seed=7, epoch=1)["anc"]
    np.testing.assert_array_equal(np.concatenate([r[0][0], r[1][0]]), a1)
    np.testing.assert_array_equal(np.concatenate([r[0][1], r[1][1]]), st[a0][a1])


def _gpu_count():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(_gpu_count() < 2, reason="needs two CUDA devices (NCCL cannot put two ranks on one GPU)")
def test_two_gpus_nccl_match_single(smc, tmp_path):
    """comm="nccl" (records through NCCL, host-batched epoch loop, CUDA-IPC
    peer stores over NVLink) is bit-identical to one process holding all
    particles: CRBD (both RNG readings), ClaDS2-LR and a configs[4] step."""
    import torch.multiprocessing as mp
    import oracle
    n_per, seed = 3000, 23
    port = dist_workers.free_port()
    mp.spawn(dist_workers.gpu_nccl_worker, args=(2, port, str(tmp_path), n_per, seed), nprocs=2, join=True)
    r = [np.load(tmp_path / f"n{k}.npy", allow_pickle=True)[0] for k in range(2)]
    t90 = inputs.tree("tree90")
    for name, m in (("crbd", smc.Model.crbd(t90)), ("crbd_lr", smc.Model.crbd(t90, lineage=True)),
                    ("clads2_lr", smc.Model.clads2(t90, lineage=True))):
        ref = smc.Smc(m, 2 * n_per, seed)
        assert ref.run_status() == r[0][name][0] == r[1][name][0] == smc.OK, name
        assert r[0][name][1] == r[1][name][1] == ref.log_z, name
        for k, get in ((2, ref.ancestors), (3, ref.log_weights), (4, ref.fields)):
            np.testing.assert_array_equal(np.concatenate([r[0][name][k], r[1][name][k]]), get(), err_msg=name)
    N = 2 * n_per
    lw = inputs.resample_lw(N, 2.0, 0.2, seed=41)
    st = inputs.state_bytes(N, 64, seed=42)
    a0 = oracle.resample(lw, seed=7, epoch=0)["anc"]
    a1 = oracle.resample(lw, seed=7, epoch=1)["anc"]
    np.testing.assert_array_equal(np.concatenate([r[0]["resample"][0], r[1]["resample"][0]]), a1)
    np.testing.assert_array_equal(np.concatenate([r[0]["resample"][1], r[1]["resample"][1]]), st[a0][a1])
