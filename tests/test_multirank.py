"""World-size-2 gloo test of the multi-GPU host logic (sharding + the single
int64 all-reduce of per-centroid statistics). The per-rank solves use the CPU
oracle here (no GPU in this container); on the B200 path bench.py runs the same
logic with the CUDA campaign and NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

WORLD = 2
PER_RANK = 96


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, out_dir):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2403_07824_b200 import distributed as D
    from tests.helpers import oracle_codebook, setup_case

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    cfg, basis, cb, _ = setup_case("C1", 64)
    K = basis["eigenvalues"].size
    index0, n = D.shard(rank, WORLD, PER_RANK)
    xi = oracle.draw_standard_normal(n, K, cfg["master_seed"], index0)
    res = oracle.run_campaign(1, cfg["mesh_resolution"], "cholesky", oracle_codebook(cb), basis["eigenvalues"],
                              basis["eigenvectors"], xi, cfg["eps"], threads=1)
    t = torch.from_numpy(D.pack_stats(res, cb["P"]))
    D.allreduce_stats(t)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_campaign_matches_single_process(tmp_path):
    from tests.helpers import oracle_codebook, setup_case
    import oracle
    from paper_2403_07824_b200 import distributed as D

    port = _free_port()
    mp.spawn(_worker, args=(port, str(tmp_path)), nprocs=WORLD, join=True)
    merged = [np.load(tmp_path / f"r{r}.npy") for r in range(WORLD)]
    assert np.array_equal(merged[0], merged[1])
    cfg, basis, cb, _ = setup_case("C1", 64)
    xi = oracle.draw_standard_normal(WORLD * PER_RANK, basis["eigenvalues"].size, cfg["master_seed"])
    ref = oracle.run_campaign(1, cfg["mesh_resolution"], "cholesky", oracle_codebook(cb), basis["eigenvalues"],
                              basis["eigenvectors"], xi, cfg["eps"])
    assert np.array_equal(merged[0], D.pack_stats(ref, cb["P"]))


def test_shard_ranges():
    from paper_2403_07824_b200 import distributed as D
    assert D.shard(1, 4, 100, index0=7) == (107, 100)
    spans = [D.split(1003, r, 4) for r in range(4)]
    assert sum(c for _, c in spans) == 1003 and spans[0][0] == 0
    assert all(spans[i][0] + spans[i][1] == spans[i + 1][0] for i in range(3))
