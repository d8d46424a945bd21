"""End-to-end operator sequences (BASELINE.json configs[4]) as reference op specs.

SURVEY.md §8d: "ResNet-50 conv/fc/pool specs: convs pre-padded, global avgpool F=7, fc as GEMM;
global batch 128. GPT-2 small: B=16, T=512, d=768, H=12 (B·H = 192 matches config B), QKV/out/MLP
GEMMs + QKᵀ/PV batched + softmax."

The reference describes single operators only (op kinds gemm, gemv, conv2d, avgpool2d,
op_spec.cpp:70-131), so a network is a sequence of operator specs, each constructed and executed
on synthetic inputs of its shape:
  * conv2d has no padding parameter (op_spec.cpp:55-60): a "same" k x k convolution is the valid
    convolution of the input pre-padded by k-1 (stride 1) or to the size that gives the output
    extent (stride 2);
  * ResNet's max-pool is expressed with the reference's avgpool2d kind (same window/stride);
  * GPT-2's layernorm/GELU/residual adds have no reference kind and are not in the sequence;
    the vocabulary projection uses the padded vocabulary 50304 (a multiple of 64).
Batch sharding over g GPUs: ResNet N/g images per GPU; GPT-2 B/g sequences per GPU
(M = B·T/g GEMM rows, B·H/g attention batches). Every op of a sequence is independent work.
"""
from __future__ import annotations

from collections import OrderedDict


def _conv(n, c, hw_in, f, k, stride):
    """Valid conv that reproduces a 'same'-padded k x k conv of an hw_in x hw_in input."""
    out = (hw_in + stride - 1) // stride if k > 1 or stride > 1 else hw_in
    padded = (out - 1) * stride + k
    return {"kind": "conv2d", "I": [n, c, padded, padded], "K": [f, c, k, k], "S": stride}


def resnet50(batch: int = 128) -> list[tuple[str, dict]]:
    """ResNet-50 v1.5 (stride on the 3x3) at 224x224: 53 convs, the stem pool, global pool, fc."""
    n = batch
    seq = [("conv1", _conv(n, 3, 224, 64, 7, 2)),
           ("pool1", {"kind": "avgpool2d", "I": [n, 64, 113, 113], "F": 3, "S": 2})]
    c_in, hw = 64, 56
    for stage, (width, blocks, stride) in enumerate([(64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)], 1):
        out_c = width * 4
        for b in range(blocks):
            s = stride if b == 0 else 1
            tag = f"layer{stage}.{b}"
            seq.append((f"{tag}.conv1", _conv(n, c_in, hw, width, 1, 1)))
            seq.append((f"{tag}.conv2", _conv(n, width, hw, width, 3, s)))
            hw_out = hw // s
            seq.append((f"{tag}.conv3", _conv(n, width, hw_out, out_c, 1, 1)))
            if b == 0:
                seq.append((f"{tag}.downsample", _conv(n, c_in, hw, out_c, 1, s)))
            c_in, hw = out_c, hw_out
    seq.append(("avgpool", {"kind": "avgpool2d", "I": [n, 2048, 7, 7], "F": 7, "S": 1}))
    seq.append(("fc", {"kind": "gemm", "M": n, "K": 2048, "N": 1000}))
    return seq


def gpt2(batch: int = 16, seq_len: int = 512, d: int = 768, heads: int = 12, layers: int = 12,
         vocab: int = 50304) -> list[tuple[str, dict]]:
    """GPT-2 small forward: per layer QKV / QK^T / softmax / PV / out-proj / MLP; then the LM head.
    GEMMs and batched attention GEMMs in bf16 (dtype_bytes 2), softmax in fp32."""
    m = batch * seq_len
    hd = d // heads
    bh = batch * heads
    layer = [
        ("qkv", {"kind": "gemm", "M": m, "K": d, "N": 3 * d, "dtype_bytes": 2}),
        ("qk", {"kind": "gemm", "M": seq_len, "K": hd, "N": seq_len, "dtype_bytes": 2, "batch": bh}),
        ("softmax", {"kind": "softmax", "M": bh * seq_len, "N": seq_len}),
        ("pv", {"kind": "gemm", "M": seq_len, "K": seq_len, "N": hd, "dtype_bytes": 2, "batch": bh}),
        ("proj", {"kind": "gemm", "M": m, "K": d, "N": d, "dtype_bytes": 2}),
        ("fc1", {"kind": "gemm", "M": m, "K": d, "N": 4 * d, "dtype_bytes": 2}),
        ("fc2", {"kind": "gemm", "M": m, "K": 4 * d, "N": d, "dtype_bytes": 2}),
    ]
    seq = [(f"h{i}.{name}", spec) for i in range(layers) for name, spec in layer]
    seq.append(("lm_head", {"kind": "gemm", "M": m, "K": d, "N": vocab, "dtype_bytes": 2}))
    return seq


SEQUENCES = {"resnet50": (resnet50, 128), "gpt2": (gpt2, 16)}


def sharded(name: str, world: int) -> list[tuple[str, dict]]:
    """The sequence for one of `world` GPUs: the global batch split evenly (batch-sharded)."""
    fn, global_batch = SEQUENCES[name]
    if global_batch % world:
        raise ValueError(f"{name}: global batch {global_batch} not divisible by {world} GPUs")
    return fn(global_batch // world)


def distinct(seq: list[tuple[str, dict]]) -> "OrderedDict[str, dict]":
    """Distinct op specs of a sequence (keyed by canonical JSON), construction happens once each."""
    import json

    out: "OrderedDict[str, dict]" = OrderedDict()
    for _, spec in seq:
        out.setdefault(json.dumps(spec, sort_keys=True), spec)
    return out
