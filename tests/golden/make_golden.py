"""Regenerate the golden fixtures in tests/golden/ (run in the container that
has /root/reference; the GPU box only reads the committed JSON).

    make -C oracle && python tests/golden/make_golden.py

Sources, by fixture:
  rng_golden.json         reference proj/tests/golden/rng_golden.json cases
                          (words + draws, the reference's own pinning data),
                          extended with draws/masks computed by the reference
                          library (oracle/_ref) at extreme keys.
  plan_golden.json        reference overlap_matrix (oracle/_ref) at the
                          BASELINE configs: entry counts, bytes moved, sha256
                          of the entry list, per-rank lane bytes.
  checksum_golden.json    no reference checksum exists: row sums for fixed
                          inputs from oracle/checksum_spec.py, the pure-Python
                          restatement of the ew_api.h spec that shares no code
                          with oracle/ew_oracle.c (the C oracle and the GPU are
                          both checked against it).
  reduce_golden.json      oracle fixed-point fold for a fixed small input.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import checksum_spec  # noqa: E402
from oracle.ew_oracle import load_oracle, load_reference  # noqa: E402
from paper_2510_00606_b200 import configs  # noqa: E402

OUT = Path(__file__).resolve().parent
REF_GOLDEN = Path("/root/reference/proj/tests/golden/rng_golden.json")


def entries_sha(rows: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(rows, dtype=np.int64).tobytes()).hexdigest()


def rng_golden(ref) -> dict:
    base = json.loads(REF_GOLDEN.read_text())
    extra = []
    keys = [(0, 2**63 + 5, 0xFFFFFFFF, 7), (2024, 1023, 31, 3), (5, 0, 1, 0),
            (2**64 - 1, 2**64 - 1, 0xFFFFFFFF, 0xFFFFFFFF)]
    for seed, sample, layer, op in keys:
        d = ref.draw(seed, sample, layer, op, 37)
        extra.append({"seed": seed, "sample": sample, "layer": layer, "op": op,
                      "draws_hex": [float(x).hex() for x in d]})
    masks = []
    for seed, lo, ns, layer, op, n, keep in [(0, 0, 3, 0, 0, 77, 0.5), (2024, 1000, 2, 5, 1, 64, 0.3),
                                             (7, 2**40, 2, 2, 9, 33, 0.9)]:
        m = ref.dropout_mask(seed, lo, ns, layer, op, n, keep)
        masks.append({"seed": seed, "sample_lo": lo, "n_samples": ns, "layer": layer, "op": op,
                      "n_elems": n, "keep": keep, "bits": m.astype(np.int64).tolist()})
    return {"source": str(REF_GOLDEN), "key_domain": base["key_domain"], "cases": base["cases"],
            "ref_draws": extra, "ref_masks": masks}


def plan_cases():
    c125, c7, c7t, c8 = (configs.gpt_125m(), configs.llama2_7b(), configs.llama2_7b_per_tensor(),
                         configs.llama3_8b())
    return [
        ("125M 4->3 drop r1", c125, list(range(4)), [0, 2, 3]),
        ("7B 8->7 drop r0", c7, list(range(8)), [1, 2, 3, 4, 5, 6, 7]),
        ("7B 8->7 drop r3", c7, list(range(8)), [0, 1, 2, 4, 5, 6, 7]),
        ("7B 8->7 drop r7", c7, list(range(8)), [0, 1, 2, 3, 4, 5, 6]),
        ("7B per-tensor 8->7 drop r3", c7t, list(range(8)), [0, 1, 2, 4, 5, 6, 7]),
        ("8B 8->6 drop r2,r5", c8, list(range(8)), [0, 1, 3, 4, 6, 7]),
        ("8B 6->8 rejoin r2,r5", c8, [0, 1, 3, 4, 6, 7], list(range(8))),
    ]


def plan_golden(ref) -> dict:
    out = []
    for name, cfg, old, new in plan_cases():
        lb = cfg.layer_bytes
        src = ref.interleaved(lb, old)
        dst = ref.interleaved(lb, new)
        failed = sorted(set(old) - set(new))
        rows, moved, _ = ref.overlap_matrix(src, dst, cfg.total_bytes, failed, old)
        egress, ingress = {}, {}
        for s, d, lo, hi, med in rows.tolist():
            if s != d:
                egress[s] = egress.get(s, 0) + hi - lo
                ingress[d] = ingress.get(d, 0) + hi - lo
        rec = {"name": name, "layer_bytes": lb, "old": old, "new": new, "failed": failed,
               "n_entries": int(len(rows)), "total_bytes_moved": int(moved),
               "sha256": entries_sha(rows), "egress": egress, "ingress": ingress}
        if len(rows) <= 64:
            rec["entries"] = rows.tolist()
        out.append(rec)
    # adjacent double failure must be rejected by the reference
    src = ref.interleaved(configs.llama3_8b().layer_bytes, list(range(8)))
    dst = ref.interleaved(configs.llama3_8b().layer_bytes, [0, 1, 4, 5, 6, 7])
    st = ref.overlap_matrix(src, dst, configs.llama3_8b().total_bytes, [2, 3], list(range(8)),
                            return_status=True)
    return {"cases": out, "adjacent_failure_status": int(st)}


def checksum_golden(orc) -> dict:
    rng = np.random.default_rng(2024)
    cases = []
    for block in (4096, 65536):
        # four segments with every local/global misalignment class
        segs, local = [], 0
        g = 3
        for length in (5, 70001, 9, 131077):
            segs.append({"global_lo": g, "length": length, "local_off": local})
            local += length
            g += length + int(rng.integers(1, 40000))
        buf = rng.integers(0, 256, size=local, dtype=np.uint8)
        rows = checksum_spec.rows_of_buffer(segs, block, buf.tobytes())
        assert rows == [int(x) for x in orc.row_sums(segs, block, buf)], "C oracle != spec"
        cases.append({"block_bytes": block, "segments": segs,
                      "buf_sha256": hashlib.sha256(buf.tobytes()).hexdigest(),
                      "buf_seed": 2024, "rows": [str(x) for x in rows]})
    synth = {}
    for seed in (0, 2024):
        s = checksum_spec.synthetic_block_sums(seed, 300_007, 65536)
        assert s == [int(x) for x in orc.block_sums_synthetic(seed, 300_007, 65536)]
        synth[str(seed)] = [str(x) for x in s]
    # synthetic state placed by a misaligned 3-segment map: rows straight
    # from the spec (GPU fill + snapshot must reproduce them)
    segs3 = [{"global_lo": 13, "length": 9001, "local_off": 0},
             {"global_lo": 70003, "length": 4, "local_off": 9001},
             {"global_lo": 131069, "length": 70000, "local_off": 9005}]
    synth_rows = {str(seed): [str(x) for x in checksum_spec.rows_of_synthetic(segs3, 4096, seed)]
                  for seed in (0, 2024)}
    return {"spec": "include/ew_api.h 'Checksum spec'; no reference implementation exists",
            "generated_by": "oracle/checksum_spec.py (independent of oracle/ew_oracle.c)",
            "cases": cases, "synthetic_300007": synth,
            "synthetic_rows": {"block_bytes": 4096, "segments": segs3, "rows": synth_rows}}


def reduce_golden(orc) -> dict:
    rng = np.random.default_rng(5)
    g = rng.normal(0, 1e-3, size=(5, 257)).astype(np.float32)
    g[1, 17] = 1e2
    g[3, 200] = -1e2
    w = np.array([7, 7, 6, 6, 6], dtype=np.float64) / 32
    amax = float(np.max(np.abs(w[:, None] * g.astype(np.float64))))
    f = orc.fixed_point_bits(amax, 5)
    acc = orc.weighted_fixed(w, g, f)
    return {"seed": 5, "weights": w.tolist(), "frac_bits": f, "absmax": amax.hex(),
            "acc_sha256": hashlib.sha256(acc.tobytes()).hexdigest(),
            "acc_head": [int(x) for x in acc[:8]]}


def main():
    orc = load_oracle()
    ref = load_reference()
    if ref is None:
        raise SystemExit("reference library not built: make -C oracle (needs /root/reference)")
    for name, fn, arg in (("rng_golden.json", rng_golden, ref), ("plan_golden.json", plan_golden, ref),
                          ("checksum_golden.json", checksum_golden, orc),
                          ("reduce_golden.json", reduce_golden, orc)):
        (OUT / name).write_text(json.dumps(fn(arg), indent=1) + "\n")
        print("wrote", OUT / name)


if __name__ == "__main__":
    main()
