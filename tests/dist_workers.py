"""Worker functions for the multi-process tests (importable by spawn)."""
import ctypes as C
import os
import socket

import numpy as np


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def init(rank, world, port, backend="gloo"):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group(backend, rank=rank, world_size=world)
    return dist


def cpu_worker(rank, world, port, outdir):
    """Host logic of the sharded path over gloo (no GPU needed)."""
    dist = init(rank, world, port)
    import paper_2112_00364_b200 as smc
    from paper_2112_00364_b200 import dist as sdist
    rng = np.random.default_rng(1000 + rank)
    # 1. each rank contributes its shard total; every rank plans the same ranges
    my_total = int(rng.integers(0, 2 ** 62)) * int(rng.integers(1, 2 ** 30))
    totals = [int(x) for x in (v for v in
              (int.from_bytes(b, "little") for b in sdist.allgather_bytes(my_total.to_bytes(16, "little"))))]
    z = 0x1234567890ABC
    plan = smc.plan_ranges(totals, 1000, z)
    # 2. the host all-gather callback used by the C library
    ag = sdist.HostAllgather()
    send = (C.c_char * 16)(*bytes([rank + 1] * 16))
    recv = (C.c_char * (16 * world))()
    rc = ag.cfunc(C.cast(send, C.c_void_p), C.cast(recv, C.c_void_p), 16, None)
    # 3. NCCL unique-id broadcast (rank 0 creates it) if NCCL loads here
    try:
        nid = sdist.nccl_unique_id()
    except Exception as e:           # NCCL not loadable on this host
        nid = repr(e).encode()
    np.save(os.path.join(outdir, f"r{rank}.npy"),
            np.array([totals, plan, list(bytes(recv)), rc, nid], dtype=object), allow_pickle=True)
    dist.destroy_process_group()


def gpu_worker(rank, world, port, outdir, n_per, seed, lineage):
    """Real sharded path: one process per shard on the same GPU, host comm
    (gloo) for the 16-byte records, CUDA IPC for particle migration."""
    dist = init(rank, world, port)
    import torch
    torch.cuda.set_device(0)
    import inputs
    import paper_2112_00364_b200 as smc
    from paper_2112_00364_b200 import dist as sdist
    m = smc.Model.crbd(inputs.tree("tree90"), lineage=lineage)
    h = sdist.ShardedSmc(m, n_per, seed, comm="host")
    rc = h.run_status()
    res = np.empty(6, dtype=object)
    res[:] = [rc, h.log_z, h.ancestors(), h.log_weights(), h.fields(), h.stats()]
    np.save(os.path.join(outdir, f"g{rank}.npy"), res, allow_pickle=True)
    h.close()
    dist.barrier()
    dist.destroy_process_group()


def gpu_resample_worker(rank, world, port, outdir, n_per):
    """configs[4] across processes on one GPU: host comm + CUDA IPC."""
    dist = init(rank, world, port)
    import torch
    torch.cuda.set_device(0)
    import inputs
    import paper_2112_00364_b200 as smc
    from paper_2112_00364_b200 import dist as sdist
    S = 64
    N = world * n_per
    lw = inputs.resample_lw(N, 2.0, 0.2, seed=41)[rank * n_per:(rank + 1) * n_per]
    st = inputs.state_bytes(N, S, seed=42)[rank * n_per:(rank + 1) * n_per]
    h = sdist.ShardedSmc(smc.Model.resample_bench(S), n_per, 7, comm="host")
    h.load(lw, smc.aos_to_soa(st).ravel())
    h.resample_step(0)
    h.resample_step(1)
    out = smc.soa_to_aos(h.state().reshape(S // 16, n_per, 16))
    res = np.empty(2, dtype=object)
    res[0], res[1] = h.ancestors(), out
    np.save(os.path.join(outdir, f"rs{rank}.npy"), res, allow_pickle=True)
    h.close()
    dist.barrier()
    dist.destroy_process_group()


def gpu_nccl_worker(rank, world, port, outdir, n_per, seed):
    """One process per GPU with comm="nccl" (the bench's multi-GPU path):
    CRBD (both RNG readings) and ClaDS2-LR runs plus a configs[4] resampling
    step; results saved for comparison with one process holding all particles."""
    dist = init(rank, world, port)
    import torch
    torch.cuda.set_device(rank)
    import inputs
    import paper_2112_00364_b200 as smc
    from paper_2112_00364_b200 import dist as sdist
    t90 = inputs.tree("tree90")
    out = {}
    for name, m in (("crbd", smc.Model.crbd(t90)), ("crbd_lr", smc.Model.crbd(t90, lineage=True)),
                    ("clads2_lr", smc.Model.clads2(t90, lineage=True))):
        h = sdist.ShardedSmc(m, n_per, seed, comm="nccl")
        rc = h.run_status()
        out[name] = [rc, h.log_z, h.ancestors(), h.log_weights(), h.fields()]
        h.close()
    S = 64
    N = world * n_per
    lw = inputs.resample_lw(N, 2.0, 0.2, seed=41)[rank * n_per:(rank + 1) * n_per]
    st = inputs.state_bytes(N, S, seed=42)[rank * n_per:(rank + 1) * n_per]
    h = sdist.ShardedSmc(smc.Model.resample_bench(S), n_per, 7, comm="nccl")
    h.load(lw, smc.aos_to_soa(st).ravel())
    h.resample_step(0)
    h.resample_step(1)
    out["resample"] = [h.ancestors(), smc.soa_to_aos(h.state().reshape(S // 16, n_per, 16))]
    h.close()
    res = np.empty(1, dtype=object)
    res[0] = out
    np.save(os.path.join(outdir, f"n{rank}.npy"), res, allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()
