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
