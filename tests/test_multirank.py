"""N > 1 host logic of bench.py on CPU: two processes over gloo (127.0.0.1), world_size 2.

The path shards by image (every image is an independent problem, no
data-path collective).  Checked here: the shards are disjoint and cover the global batch in
order; processing each shard on its own rank and concatenating gives exactly the
single-process result (oracle pipeline, so no GPU is needed); the step time is the MAX over
ranks and the reported value is the whole job's pixels over that time.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import oracle
import synth

CFG, B_PER_RANK, WORLD = "C5", 2, 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, outdir: str) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        first, n = bench.shard(world, rank, B_PER_RANK)
        x = synth.make_config(CFG, batch=n, first=first, threads=1)
        r = oracle.enhance_batch(x, oracle.Params(), nthreads=1, want_out=True)
        ms = bench.max_over_ranks(1.0 + 0.5 * rank, dist, torch.device("cpu"))  # rank 1 is slower
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), first=first, n=n, x=x, out=r["out"], lut=r["lut"],
                 ms=ms)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def ranks(tmp_path_factory):
    d = str(tmp_path_factory.mktemp("mr"))
    mp.spawn(_worker, args=(WORLD, _free_port(), d), nprocs=WORLD, join=True)
    return [dict(np.load(os.path.join(d, f"rank{r}.npz"))) for r in range(WORLD)]


def test_shards_disjoint_and_cover(ranks):
    spans = [(int(r["first"]), int(r["n"])) for r in ranks]
    assert spans == [(0, B_PER_RANK), (B_PER_RANK, B_PER_RANK)]
    full = synth.make_config(CFG, batch=WORLD * B_PER_RANK, threads=1)
    assert np.array_equal(np.concatenate([r["x"] for r in ranks]), full)


def test_sharded_equals_single_process(ranks):
    full = synth.make_config(CFG, batch=WORLD * B_PER_RANK, threads=1)
    ref = oracle.enhance_batch(full, oracle.Params(), nthreads=2, want_out=True)
    assert np.array_equal(np.concatenate([r["out"] for r in ranks]), ref["out"])
    assert np.array_equal(np.concatenate([r["lut"] for r in ranks]), ref["lut"])


def test_step_time_is_max_over_ranks(ranks):
    assert [float(r["ms"]) for r in ranks] == [1.5, 1.5]


def test_aggregate_value_counts_every_rank():
    c = synth.CONFIGS[CFG]
    one = bench.aggregate_mps(1, c.B, c.H, c.W, 1.0)
    assert bench.aggregate_mps(2, c.B, c.H, c.W, 1.0) == pytest.approx(2 * one)
    assert one == pytest.approx(c.B * c.H * c.W / 1e-3 / 1e6)


def test_shard_rejects_bad_rank():
    with pytest.raises(AssertionError):
        bench.shard(2, 2, 4)
