"""The N>1 path on CPU: input sharding + output all_gather across 2 gloo ranks.

Each rank computes its contiguous block of inputs (here with the oracle, since
there is no GPU in this container — the per-rank compute is the same call the
GPU ranks make) and the gathered result must equal the single-process result
bit for bit, including uneven shards."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_04779_b200.sharding import gather_outputs, shard_range


def test_shard_range_partitions():
    for B in (1, 2, 5, 32, 320, 321):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_range(B, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == B
            for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
                assert a1 == b0
            sizes = [b1 - b0 for b0, b1 in ranges]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, x, result_path):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "tests")]
    import oracle as O
    from cases import make_case

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p, Y, H = make_case(2, 16, 8, 9, B, x, 5, 6)
    b0, b1 = shard_range(B, rank, world)
    local = O.el_layer_step(p, Y[b0 * x:b1 * x], H[b0:b1], x)   # this rank's inputs only
    full = gather_outputs(torch.from_numpy(local), B, x)
    if rank == 0:
        np.save(result_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [4, 5])
def test_two_rank_gloo_gather_matches_single_process(tmp_path, B):
    import oracle as O
    from cases import make_case

    x = 3
    out_path = str(tmp_path / "full.npy")
    mp.start_processes(_worker, args=(2, _free_port(), B, x, out_path), nprocs=2, join=True, start_method="spawn")
    p, Y, H = make_case(2, 16, 8, 9, B, x, 5, 6)
    want = O.el_layer_step(p, Y, H, x)
    assert np.array_equal(np.load(out_path), want)


def test_bench_spawns_ranks_and_checks_shards():
    """`bench.py --gpus 2` outside torchrun starts its 2 ranks itself (torch.distributed.run),
    shards the inputs, takes the max over ranks, all_gathers the outputs and has rank 0
    recompute rank 1's shard bit for bit — here over gloo with the CPU stand-in for the
    kernels (ELATTN_BENCH_STANDIN=cpu), the same plumbing the GPU arm runs over NCCL."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, ELATTN_BENCH_STANDIN="cpu")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1",
                        "--batch", "3", "--layers", "2"], capture_output=True, text=True, timeout=600, cwd=root,
                       env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["global_batch"] == 6 and line["value"] > 0
    assert line["shard_check"] == {"ranks_recomputed_on_rank0": [1], "bit_exact": True, "rows_per_rank": 12}
