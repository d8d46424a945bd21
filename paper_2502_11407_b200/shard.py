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


# Variants whose program does more tensor work than the `auto` one the cost model prices:
# 3xTF32 issues three tf32 UMMAs per product (measured 2.4x the tf32 GEMM on config G).
VARIANT_WORK = {"tc_3xtf32": 3.0}


def estimated_seconds(op_docs: Sequence[dict], hw, variants: Sequence[str] | None = None) -> list[float]:
    """The engine's predicted time of the program `auto` runs for the best B200-mode schedule of
    every op (cost `exec_seconds`: the tensor-core / HBM-streaming / SIMT program; the LPT weights)."""
    import paper_2502_11407_b200 as g

    out = []
    for i, doc in enumerate(op_docs):
        op = g.TensorOpSpec.parse_text(json.dumps(doc))
        res = g.optimize(op, hw, g.EngineConfig(mode="b200", top_k=1))
        cost = res[0]["cost"]
        scale = VARIANT_WORK.get(variants[i], 1.0) if variants else 1.0
        out.append(scale * float(cost.get("exec_seconds", cost["est_seconds"])))  # batch-aware already
    return out


def suite_partition(op_docs: Sequence[dict], hw, world: int, variants: Sequence[str] | None = None) -> list[list[int]]:
    return lpt(estimated_seconds(op_docs, hw, variants), world)
