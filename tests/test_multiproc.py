"""Multi-process (world_size 2, gloo on CPU) checks of the multi-GPU driver logic: the suite LPT
partition and the batch-sharded sequences divide the work exactly, every rank derives the same
partition, and the max-over-ranks timing reduction / result gather behave as bench.py uses them.
No collective is on the compute path; these are the only torch.distributed calls the driver makes."""
import json
import os
import sys

import pytest

torch = pytest.importorskip("torch")
dist = pytest.importorskip("torch.distributed")
mp = pytest.importorskip("torch.multiprocessing")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SUITE = [
    {"kind": "gemm", "M": 1024, "K": 1024, "N": 1024},
    {"kind": "gemm", "M": 512, "K": 64, "N": 512, "dtype_bytes": 2, "batch": 192},
    {"kind": "gemv", "M": 32768, "N": 4096},
    {"kind": "softmax", "M": 32768, "N": 4096},
    {"kind": "dwconv2d", "I": [32, 256, 114, 114], "K": [256, 1, 3, 3], "S": 1},
    {"kind": "avgpool2d", "I": [32, 256, 114, 114], "F": 3, "S": 1},
    {"kind": "conv2d", "I": [16, 64, 58, 58], "K": [64, 64, 3, 3], "S": 1},
]


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2502_11407_b200 as g
    from paper_2502_11407_b200 import sequences as S, shard
    from test_sequences import B200_DOC

    hw = g.HardwareSpec.load_text(json.dumps(B200_DOC))
    parts = shard.suite_partition(SUITE, hw, world)
    mine = parts[rank]
    # every rank derives the same partition
    gathered = [None] * world
    dist.all_gather_object(gathered, parts)
    same = all(p == parts for p in gathered)
    # batch sharding: this rank's GPT-2 shard
    f_mine = sum(g.TensorOpSpec.parse_text(json.dumps(s)).flops for _, s in S.sharded("gpt2", world))
    f_all = torch.tensor([f_mine], dtype=torch.float64)
    dist.all_reduce(f_all)
    # timing reduction as bench.py does it: max over ranks
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    q.put((rank, mine, same, f_all.item(), t.item()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_partition_and_reductions(world):
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    units = sorted(i for _, mine, _, _, _ in res for i in mine)
    assert units == list(range(len(SUITE)))            # every op exactly once
    assert all(same for _, _, same, _, _ in res)       # identical partition on every rank
    sys.path.insert(0, ROOT)
    import paper_2502_11407_b200 as g
    from paper_2502_11407_b200 import sequences as S

    f_global = sum(g.TensorOpSpec.parse_text(json.dumps(s)).flops for _, s in S.sharded("gpt2", 1))
    for _, _, _, f_sum, t_max in res:
        assert abs(f_sum - f_global) <= 1e-9 * f_global  # the shards add up to the global batch
        assert t_max == float(world)                     # max over ranks


def test_lpt_balances():
    sys.path.insert(0, ROOT)
    from paper_2502_11407_b200 import shard

    costs = [7, 5, 4, 3, 3, 2, 2, 1]
    bins = shard.lpt(costs, 3)
    loads = sorted(sum(costs[i] for i in b) for b in bins)
    assert sorted(i for b in bins for i in b) == list(range(len(costs)))
    assert loads[-1] - loads[0] <= max(costs)
    assert shard.lpt(costs, 1) == [list(range(len(costs)))]
    with pytest.raises(ValueError):
        shard.lpt(costs, 0)
