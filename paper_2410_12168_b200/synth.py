"""Seeded synthetic inputs for the W4Ax path (shared by tests and bench).

This module holds none of the method's arithmetic: it only draws random
numbers and builds the layer's calibration artefact (permutation + block
mask) from outlier positions it planted itself.  Both the CUDA path and the
CPU oracle consume exactly the bytes produced here.

Recipe:
  * X ~ N(0, 1), rounded to fp16 (RNE).
  * For each INT8 block, ``outliers_per_block`` (default 32) of its channels
    are outlier channels: a seeded random ORIGINAL channel position whose
    column is scaled by a gain gamma ~ log-uniform[10, 100] -- "magnitudes
    that can exceed typical hidden state values by tenfold or even a
    hundredfold" (§3.1), confined to specific channels.
  * The permutation perm[new] = old moves the planted outlier channels into
    the INT8 blocks (§3.2 "cluster these channels into a single
    block"); ordering: outliers by descending gain (ties: ascending index),
    the rest stable.
  * W ~ N(0, 1/K), rounded to fp16 (so |Y| stays well inside fp16 range).
  * block_bits: K/128 entries, 8 for INT8 blocks, 4 otherwise.  ``mask``
    chooses where the INT8 blocks sit: "prefix" (blocks 0..n8-1, the layout
    a permutation produces), "scattered" (evenly spread), or an explicit list.
"""
from __future__ import annotations

import numpy as np

BLOCK = 128


def block_bits_for(K: int, n8: int, mask="prefix", k: int = BLOCK) -> np.ndarray:
    nb = K // k
    bits = np.full(nb, 4, np.uint8)
    if isinstance(mask, (list, tuple, np.ndarray)):
        bits[:] = np.asarray(mask, dtype=np.uint8)
        return bits
    if n8 <= 0:
        return bits
    if mask == "prefix":
        bits[:n8] = 8
    elif mask == "scattered":
        idx = np.unique(np.linspace(0, nb - 1, n8).round().astype(int))
        bits[idx] = 8
    else:
        raise ValueError(mask)
    return bits


def make_problem(M: int, N: int, K: int, n8: int = 0, seed: int = 0, mask="prefix",
                 outliers_per_block: int = 32, with_perm: bool = True, k: int = BLOCK,
                 x_rows=None):
    """Build one seeded W4Ax problem.

    Returns dict(X fp16 [M x K] or [len(x_rows) x K], W fp16 [N x K],
    perm int32 [K] or None, bits uint8 [K/k], outlier_channels, gains)."""
    rng = np.random.default_rng(seed)
    bits = block_bits_for(K, n8, mask, k)
    int8_blocks = np.flatnonzero(bits == 8)
    n_out = int(min(outliers_per_block, k) * len(int8_blocks))
    out_ch = np.sort(rng.choice(K, size=n_out, replace=False)) if n_out else np.zeros(0, np.int64)
    gains = np.exp(rng.uniform(np.log(10.0), np.log(100.0), size=n_out))

    perm = None
    if with_perm:
        # outliers first by descending gain (ties ascending index), rest stable
        order = np.lexsort((out_ch, -gains))
        out_sorted = out_ch[order]
        is_out = np.zeros(K, bool)
        is_out[out_ch] = True
        normal = np.flatnonzero(~is_out)
        # lay the outlier channels into the INT8 blocks (in block order),
        # the normal channels fill every remaining position in order
        perm = np.full(K, -1, np.int64)
        per_blk = min(outliers_per_block, k)
        pos = []
        for b in int8_blocks:
            pos.extend(range(b * k, b * k + per_blk))
        pos = np.asarray(pos, dtype=np.int64)
        perm[pos] = out_sorted
        perm[perm < 0] = normal
        perm = perm.astype(np.int32)

    col_gain = np.ones(K, np.float32)
    col_gain[out_ch] = gains.astype(np.float32)

    rows = M if x_rows is None else len(x_rows)
    X = rng.standard_normal((M, K), dtype=np.float32) if x_rows is None else None
    if X is None:
        # regenerate the full stream so sampled rows equal the full problem's rows
        X = rng.standard_normal((M, K), dtype=np.float32)[np.asarray(x_rows)]
    X *= col_gain[None, :]
    W = (rng.standard_normal((N, K), dtype=np.float32) * np.float32(1.0 / np.sqrt(K)))
    return {
        "X": X.astype(np.float16),
        "W": W.astype(np.float16),
        "perm": perm,
        "bits": bits,
        "outlier_channels": out_ch,
        "gains": gains,
        "M": rows, "N": N, "K": K,
    }


def sample_rows(M: int, count: int = 64, seed: int = 0) -> np.ndarray:
    """Fixed row sample for large-M parity: first, last, seeded random."""
    if M <= count:
        return np.arange(M, dtype=np.int32)
    rng = np.random.default_rng(seed + 7919)
    mid = rng.choice(np.arange(1, M - 1), size=count - 2, replace=False)
    return np.sort(np.concatenate([[0, M - 1], mid])).astype(np.int32)
