"""The multi-process row-sharded path (mode 2: one process per rank, CUDA IPC peer memory,
device mailboxes) executed for real: two processes on the one B200 of this pool, their setup
exchanges through torch.distributed (gloo) via scg_host_comm, with sync_collectives = 1 so that the
ranks meet on the host before every device collective and no kernel ever waits for another rank's
kernel (B200_PROFILING.md: ranks whose kernels wait on one another must not share a GPU).

Every iterate is compared with the CPU oracle: the iteration records bitwise, each rank's rows of
z / y bitwise, the reconstruction, objective and feasibility to the BASELINE tolerances and the
rounded cut identically."""
import os
import tempfile

import numpy as np
import pytest

import oracle
import scg_inputs as si

pytestmark = pytest.mark.gpu


def _rank(rank, world, port, cfg, T, R, seed, outdir):
    import torch
    import torch.distributed as dist
    import paper_1912_02949_b200 as scg
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        L = si.laplacian(cfg) if cfg != "star" else _star()
        sp = scg.row_splits(L.row_ptr, world)
        g = scg.SketchyCGAL(L, R=R, seed=seed, rank=rank, world=world, splits=sp,
                            host_comm=scg.TorchHostComm(sync_collectives=True))
        g.step(T)
        log = g.iter_log()
        z, y = g.state("z"), g.state("y")
        U, lam, _ = g.reconstruct()
        obj, feas = g.objective(), g.feasibility()
        chi, w = g.round()
        g.close()
        np.savez(os.path.join(outdir, f"r{rank}.npz"), log=log, z=z, y=y, lam=lam, obj=obj, feas=feas, chi=chi,
                 w=w, a=sp[rank], b=sp[rank + 1])
    finally:
        dist.barrier()
        dist.destroy_process_group()


def _star():
    n = 3000
    return si.laplacian_from_edges(n, np.zeros(n - 50, dtype=np.int64), np.arange(1, n - 49), np.ones(n - 50))


@pytest.mark.parametrize("cfg,T,R,seed", [("c0", 60, 10, 0), ("c1", 40, 10, 1), ("star", 20, 5, 9)])
def test_two_processes_mode2_bitwise_vs_oracle(gpu, cfg, T, R, seed):
    import torch.multiprocessing as mp
    gpu.build()
    L = si.laplacian(cfg) if cfg != "star" else _star()
    world = 2
    port = 33500 + (os.getpid() % 2000)
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_rank, args=(world, port, cfg, T, R, seed, td), nprocs=world, join=True)
        res = [dict(np.load(os.path.join(td, f"r{r}.npz"))) for r in range(world)]
    o = oracle.Oracle(L, R, seed=seed, logcap=T)
    o.step(T)
    for r in res:
        np.testing.assert_array_equal(r["log"][:, [0, 1, 2, 3, 7, 8, 10, 11]], o.log[:, [0, 1, 2, 3, 7, 8, 10, 11]])
        np.testing.assert_allclose(r["log"][:, 4:7], o.log[:, 4:7], rtol=1e-13, atol=0)
        a, b = int(r["a"]), int(r["b"])
        np.testing.assert_array_equal(r["z"], o.z[a:b])
        np.testing.assert_array_equal(r["y"], o.y[a:b])
    Uo, lam_o, _ = oracle.nystrom_reconstruct(o.S, o.Omega, o.tau)
    lam_tc = oracle.trace_correct(lam_o, o.alpha) * (L.n / o.alpha)
    obj_o = oracle.objective_hat(L, Uo, lam_tc)
    f_o = oracle.feasibility_hat(Uo, lam_tc)
    chi_o, w_o, _ = oracle.round_cut(L, Uo)
    for r in res:
        np.testing.assert_allclose(r["lam"], lam_tc, rtol=1e-9)
        assert abs(r["obj"][1] - obj_o) <= 1e-6 * abs(obj_o)
        assert abs(r["feas"][1] - f_o[0]) <= 1e-6 * f_o[0]
        assert abs(float(r["w"]) - w_o) <= 1e-9 * w_o
    chi = np.concatenate([res[0]["chi"], res[1]["chi"]])
    np.testing.assert_array_equal(chi, chi_o)
