"""Toy consistency run on the B200 recovery path.

The reference's end-to-end criterion for this path is its toy simulator
test: an elastic run that loses a DP rank mid-run must end with the same
parameters as the static run, bit for bit (test_sim.cpp:136-147,
run_consistency_pair verify.cpp:55-78), and a wrongly weighted gradient
must be caught (test_sim.cpp:149-158).  The toy step is sim.cpp:895-953:

  for every global sample s of the step (its micro-batch slot's contiguous
  range, dataflow.cpp:30-40) and layer l = 1..L:
      u = draw({seed, s, l, 0}, K)                     (rng.cpp:38-53)
      g[k] = ((s+1)(l+1)(k+1) mod 7 - 3) * (u[k] < keep ? 0 : 1/keep)
  grad = sum over samples in ascending order;  params -= lr * grad / B

Here each DP rank (one per GPU, or emulated side by side on one) runs the
same step through the B200 kernels: its keep-bits come from the Philox mask
kernel keyed by global sample id (ew_philox_dropout_mask), its samples are
folded into an int64 fixed-point accumulator with weight 1/B
(ew_weighted_fold), the ranks' accumulators are summed — an exact integer
sum (NCCL int64 all-reduce on a real group) — dequantised to fp64
(ew_fixed_to_double) and applied.  After a departure the survivors take
the reshaped micro-batches (reshard_microbatches, dataflow.cpp:52-69).
Integer sums make the result independent of which rank folded which sample,
and the toy's values are dyadic, so it also equals the reference's fp64
fold exactly.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Tuple

import torch

from . import device as dev
from .fabric import reshard_microbatches, sample_ranges


@dataclass
class ToyConfig:
    """The reference's "toy" preset (presets.cpp:98-113, ToyModelConfig
    presets.hpp:29-35): DP 8, micro-batch size 1, global batch 16 (two
    micro-batches of 8), 4 layers of 4 parameters, lr 0.25, keep 0.5."""
    seed: int = 2024
    dp: int = 8
    layers: int = 4
    params_per_layer: int = 4
    microbatch_size: int = 1
    global_batch: int = 16
    learning_rate: float = 0.25
    keep_probability: float = 0.5
    steps: int = 4

    @property
    def num_microbatches(self) -> int:
        return self.global_batch // (self.dp * self.microbatch_size)

    @property
    def n_params(self) -> int:
        return self.layers * self.params_per_layer


def sample_gradients(cfg: ToyConfig, lo: int, hi: int) -> torch.Tensor:
    """Per-sample toy gradients of global samples [lo, hi): [hi-lo, L*K]
    fp32 (exact: values in {-3..3} x {0, 1/keep})."""
    n, K = hi - lo, cfg.params_per_layer
    s = torch.arange(lo, hi, dtype=torch.int64, device="cuda")[:, None]
    k = torch.arange(K, dtype=torch.int64, device="cuda")[None, :]
    cols = []
    for layer in range(1, cfg.layers + 1):
        bits = dev.dropout_mask(cfg.seed, lo, n, layer, 0, K, cfg.keep_probability)
        word = bits.to(torch.int64)[:, (k[0] // 32)] & 0xFFFFFFFF
        kept = (word >> (k % 32)) & 1
        base = ((s + 1) * (layer + 1) * (k + 1)) % 7 - 3
        cols.append(base.to(torch.float64) * kept.to(torch.float64) / cfg.keep_probability)
    return torch.cat(cols, dim=1).to(torch.float32)


def rank_sample_ranges(cfg: ToyConfig, per_slot_mbs: Sequence[int], slot_index: int,
                       step: int) -> List[Tuple[int, int]]:
    """The global sample ranges one slot consumes in a step (every
    micro-batch; the gating column tail beyond the step's batch is dropped,
    sim.cpp:913)."""
    base = step * cfg.global_batch
    out = []
    for mb in range(cfg.num_microbatches):
        lo, hi = sample_ranges(per_slot_mbs, base, mb)[slot_index]
        hi = min(hi, base + cfg.global_batch)
        if hi > lo:
            out.append((lo, hi))
    return out


def frac_bits(cfg: ToyConfig) -> int:
    """Fixed-point bits from the step's largest |w g| (1/keep * 3 / B) and
    its unit count: the same for every split of the batch."""
    absmax = 3.0 / cfg.keep_probability / cfg.global_batch
    return dev.fixed_point_bits(absmax, cfg.global_batch)


def fold_rank(cfg: ToyConfig, ranges: Sequence[Tuple[int, int]], f: int) -> torch.Tensor:
    """One rank's int64 accumulator of its samples' gradients, weight 1/B."""
    acc = torch.zeros(cfg.n_params, dtype=torch.int64, device="cuda")
    first = True
    for lo, hi in ranges:
        g = sample_gradients(cfg, lo, hi)
        units = [g[i] for i in range(g.shape[0])]
        dev.weighted_fold(units, [1.0 / cfg.global_batch] * len(units), f, acc,
                          accumulate=not first)
        first = False
    return acc


class ToyRun:
    """Static or elastic toy run.  `events`: {step: departed slots} applied
    before that step (the reference lands its failure inside step 1 and
    recovers before step 2).  Emulated (my_slots=None): every member's
    accumulator is folded on this GPU and summed there.  Distributed: each
    process passes its own slots and `reduce(acc, members)`, which sums the
    members' accumulators in place (NCCL int64 all-reduce on the current —
    after a departure, shrunk — communicator); a process whose slots all
    departed stops at the departure."""

    def __init__(self, cfg: ToyConfig, events: Optional[dict] = None,
                 inject_wrong_weights: bool = False):
        self.cfg = cfg
        self.events = dict(events or {})
        self.inject = inject_wrong_weights
        # initial toy parameters as the reference sets them (sim.cpp:429-432)
        l = torch.arange(cfg.layers, dtype=torch.float64)[:, None]
        k = torch.arange(cfg.params_per_layer, dtype=torch.float64)[None, :]
        self.params = (0.5 + 0.25 * l - 0.125 * k).reshape(-1).cuda()
        self.members = list(range(cfg.dp))
        self.per_slot_mbs = [cfg.microbatch_size] * cfg.dp
        self.consumed: List[List[int]] = []

    def _apply_events(self, step: int) -> None:
        gone = self.events.get(step)
        if gone:
            survivors = [m for m in self.members if m not in gone]
            # reshaper over slot indices of the current member list
            idx = [self.members.index(m) for m in survivors]
            _, mbs = reshard_microbatches(self.per_slot_mbs, self.cfg.num_microbatches, idx)
            self.members, self.per_slot_mbs = survivors, mbs

    def run(self, reduce: Optional[Callable] = None, my_slots: Optional[Sequence[int]] = None):
        cfg, f = self.cfg, frac_bits(self.cfg)
        for step in range(cfg.steps):
            self._apply_events(step)
            mine = [m for m in self.members if my_slots is None or m in my_slots]
            if my_slots is not None and not mine:
                break  # this process's slots left the group
            total = torch.zeros(cfg.n_params, dtype=torch.int64, device="cuda")
            seen = []
            for m in mine:
                ranges = rank_sample_ranges(cfg, self.per_slot_mbs, self.members.index(m), step)
                seen.extend(s for lo, hi in ranges for s in range(lo, hi))
                total += fold_rank(cfg, ranges, f)
            if reduce is not None:
                reduce(total, list(self.members))
            self.consumed.append(sorted(seen))
            grad = dev.fixed_to_double(total, f)
            if self.inject and len(self.members) < cfg.dp:
                # the reference's fixture (sim.cpp:940-947): stage-1 layers
                # mis-scaled by the surviving slot fraction; here the first
                # half of the layers
                bad = len(self.members) / cfg.dp
                grad[:cfg.n_params // 2] *= bad
            self.params -= cfg.learning_rate * grad
        torch.cuda.synchronize()
        return self.params
