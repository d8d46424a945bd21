"""Multi-GPU work division for the benchmark driver.

The hot path shards with no exchange step:
  * the operator suite: every (op, variant) is an independent unit; units are dealt to GPUs by
    longest-processing-time-first on the B200-mode cost estimate (`estimate_b200`), so each GPU
    gets a near-equal share of the predicted time;
  * the end-to-end sequences: the global batch is split evenly (paper_2502_11407_b200.sequences).
One process per GPU; torch.distributed is used only for the start barrier, the max-over-ranks
reduction of the timed region and gathering per-op results on rank 0 — never on the compute path.
"""
from __future__ import annotations

import heapq
import json
from typing import Sequence


def lpt(costs: Sequence[float], world: int) -> list[list[int]]:
    """Longest-processing-time-first: indices of `costs` dealt to `world` bins, each unit to the
    currently lightest bin; ties broken by index so every rank computes the same partition."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    heap = [(0.0, r) for r in range(world)]
    bins: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        bins[r].append(i)
        heapq.heappush(heap, (load + float(costs[i]), r))
    return [sorted(b) for b in bins]


def estimated_seconds(op_docs: Sequence[dict], hw) -> list[float]:
    """The engine's own cost of the best B200-mode schedule for every op (the LPT weights)."""
    import paper_2502_11407_b200 as g

    out = []
    for doc in op_docs:
        op = g.TensorOpSpec.parse_text(json.dumps(doc))
        res = g.optimize(op, hw, g.EngineConfig(mode="b200", top_k=1))
        out.append(float(res[0]["cost"]["est_seconds"]))  # batch-aware already
    return out


def suite_partition(op_docs: Sequence[dict], hw, world: int) -> list[list[int]]:
    return lpt(estimated_seconds(op_docs, hw), world)
