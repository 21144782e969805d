"""Second, independent restatement of the per-block checksum (TEST
INFRASTRUCTURE — only tests/ and tests/golden/make_golden.py import it).

The reference has no checksum (its snapshot is a timeline model,
param_fabric.hpp:86-96, param_fabric.cpp:136-142), so parity for kernel (a)
rests on a written spec.  oracle/ew_oracle.c restates that spec in C for
speed; this module restates it again, straight from the text in
include/ew_api.h ("Checksum spec"), in plain Python integers, sharing no code,
no loop structure and no arithmetic shortcut with the C oracle or the CUDA
kernels (no running sums, no word-shift decomposition, no row/segment
geometry reuse).  The golden file tests/golden/checksum_golden.json is
generated from THIS module; the C oracle and the GPU are both checked
against it.

Spec (ew_api.h):
  * the flat byte space is cut into blocks of B bytes (B a power of two);
  * global word i is bytes [8i, 8i+8) read little-endian, a byte the buffer
    does not hold reading as 0;
  * s0(b) = sum w_i and s1(b) = sum (i+1) * w_i, mod 2^64, over the words i
    of block b;
  * a "row" is one (segment, block) pair: the sums over block b's words with
    only that segment's bytes present.
Synthetic state: word i = splitmix64(seed ^ i), the published
SplitMix64 finaliser (Steele, Lea, Flood 2014; the java.util.SplittableRandom
constants).
"""
from __future__ import annotations

from typing import Callable, Dict, Iterable, List, Sequence, Tuple

MASK = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """SplitMix64 output function applied to state x (one step from x)."""
    z = (x + 0x9E3779B97F4A7C15) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def synthetic_byte(seed: int, g: int) -> int:
    """Byte at global position g of the synthetic state."""
    return (splitmix64((seed ^ (g // 8)) & MASK) >> (8 * (g % 8))) & 0xFF


def _sums_of_bytes(present: Dict[int, int]) -> Dict[int, Tuple[int, int]]:
    """Per word index: (w, (i+1) w) from a {global byte -> value} map."""
    words: Dict[int, int] = {}
    for g, v in present.items():
        words[g // 8] = words.get(g // 8, 0) | (v << (8 * (g % 8)))
    return {i: (w, ((i + 1) * w) & MASK) for i, w in words.items()}


def block_sums(present: Dict[int, int], block_bytes: int) -> Dict[int, Tuple[int, int]]:
    """{block -> (s0, s1)} of the bytes in `present` ({global byte: value})."""
    out: Dict[int, Tuple[int, int]] = {}
    words_per_block = block_bytes // 8
    for i, (a, b) in _sums_of_bytes(present).items():
        blk = i // words_per_block
        s0, s1 = out.get(blk, (0, 0))
        out[blk] = ((s0 + a) & MASK, (s1 + b) & MASK)
    return out


def rows(segments: Sequence[dict], block_bytes: int,
         byte_at: Callable[[int, int], int]) -> List[int]:
    """Row sums, flattened [s0, s1, s0, s1, ...] in row order: segments in the
    given (ascending) order, blocks ascending within a segment, empty
    segments owning no row.  byte_at(global_pos, local_pos) gives a byte."""
    out: List[int] = []
    for s in segments:
        g0, n, l0 = int(s["global_lo"]), int(s["length"]), int(s["local_off"])
        if n <= 0:
            continue
        first, last = g0 // block_bytes, (g0 + n - 1) // block_bytes
        for blk in range(first, last + 1):
            lo = max(g0, blk * block_bytes)
            hi = min(g0 + n, (blk + 1) * block_bytes)
            present = {g: byte_at(g, l0 + (g - g0)) for g in range(lo, hi)}
            s0, s1 = block_sums(present, block_bytes).get(blk, (0, 0))
            out += [s0, s1]
    return out


def rows_of_buffer(segments: Sequence[dict], block_bytes: int, buf: bytes) -> List[int]:
    """Rows of a packed shard buffer (local byte x of segment k is
    buf[local_off_k + x])."""
    return rows(segments, block_bytes, lambda g, x: buf[x])


def rows_of_synthetic(segments: Sequence[dict], block_bytes: int, seed: int) -> List[int]:
    return rows(segments, block_bytes, lambda g, x: synthetic_byte(seed, g))


def synthetic_block_sums(seed: int, total_bytes: int, block_bytes: int) -> List[int]:
    """Whole-space block sums [s0, s1, ...] of the synthetic state over
    [0, total_bytes) (the tail of the last word reads as 0)."""
    n_blocks = (total_bytes + block_bytes - 1) // block_bytes
    out = [0] * (2 * n_blocks)
    for i in range((total_bytes + 7) // 8):
        w = splitmix64((seed ^ i) & MASK)
        keep = min(8, total_bytes - 8 * i)
        if keep < 8:
            w &= (1 << (8 * keep)) - 1
        blk = (8 * i) // block_bytes
        out[2 * blk] = (out[2 * blk] + w) & MASK
        out[2 * blk + 1] = (out[2 * blk + 1] + (i + 1) * w) & MASK
    return out


def combine(parts: Iterable[Dict[int, Tuple[int, int]]]) -> Dict[int, Tuple[int, int]]:
    """Sum block-sum maps mod 2^64 (linearity: rows of any layout add up to
    the block sums of the whole space)."""
    out: Dict[int, Tuple[int, int]] = {}
    for p in parts:
        for blk, (a, b) in p.items():
            s0, s1 = out.get(blk, (0, 0))
            out[blk] = ((s0 + a) & MASK, (s1 + b) & MASK)
    return out
