"""Generate the bench workload fixtures by RUNNING THE REFERENCE.

Run in the dev container only (``/root/reference`` does not exist on the GPU
box):  ``python tests/golden/make_workload.py``.  Writes
``tests/golden/workload_<cfg>.npz`` for cfg1-cfg5: the per-query inputs of the
config path and the reference's own decisions on them.

Inputs, per query, drawn from one ``random.Random(SEED)`` stream:
* the hidden truth ``TruthDistribution(...).sample(rng)`` (workload.py:61-81)
  and the profile ``mock_estimate(truth, NoiseParams(), seed=...)``
  (profiler.py:257-309) — the default noise corrupts a field in ~4.9% of the
  queries, which then carry a low confidence and take the gate's hull;
  cfg3 builds ``QueryProfile(complex, joint, pieces ~ U[1,10], [30, 200])``
  directly;
* ``query_token_len ~ U(DATASET_PROFILES[...].input_range)`` (workload.py:53-58);
* ``free_bytes ~ U[0, 2 * the largest candidate of the gated space]`` (A2 mix,
  test_acceptance.py:186-190); cfg5: ``16 GiB - U[0, 16 GiB]`` over the full
  space {RR, ST, MR} x [1, 35] x [30, 200].

Expected outputs, from the reference itself (``oracle/refpath.py``): the gated
space and gate-fallback flag of every query (fresh window, in order), and
the decision best_fit_select -> fallback_config -> MustQueue with its plan bytes.
"""

from __future__ import annotations

import os
import random
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import refpath  # noqa: E402

SEED = 1  # seed 0 for data, 1 for queries / profiles
GiB = 1024 ** 3
CFGS = {
    "cfg1": dict(nq=1000, truth={}, lengths="single_hop_qa", chunk=1000),
    "cfg2": dict(nq=10_000, truth=dict(p_complex_given_joint=0.0, p_complex_given_simple=0.0),
                 lengths="single_hop_qa", chunk=1000),
    "cfg3": dict(nq=10_000, truth=None, lengths="multihop_qa", chunk=1000),
    "cfg4": dict(nq=8192, truth={}, lengths="doc_level_qa", chunk=1024),
    "cfg5": dict(nq=100_000, truth={}, lengths="single_hop_qa", chunk=1000, full_space=True),
}


def make(name: str, rs) -> dict:
    c = CFGS[name]
    T, M, P, W, Mem = rs.types, rs.mapping, rs.profiler, rs.workload, rs.memory
    rng = random.Random(SEED * 1000 + int(name[-1]))
    lp = W.DATASET_PROFILES[c["lengths"]]
    td = W.TruthDistribution(**c["truth"]) if c["truth"] is not None else None
    n = c["nq"]
    cols = {k: np.zeros(n, dtype=t) for k, t in (("cx", np.uint8), ("joint", np.uint8), ("pieces", np.uint16),
                                                 ("s_lo", np.uint16), ("s_hi", np.uint16), ("conf", np.float64),
                                                 ("qlen", np.int32), ("free", np.int64))}
    for i in range(n):
        if td is not None:
            truth = td.sample(rng)
            prof = P.mock_estimate(truth, P.NoiseParams(), seed=rng.getrandbits(63)).profile
        else:
            prof = M.QueryProfile(complexity_high=True, needs_joint_reasoning=True,
                                  pieces_required=rng.randint(1, 10), summary_len_range=T.IntRange(30, 200),
                                  confidence=P.CLEAN_CONFIDENCE)
        cols["cx"][i], cols["joint"][i] = prof.complexity_high, prof.needs_joint_reasoning
        cols["pieces"][i] = prof.pieces_required
        cols["s_lo"][i], cols["s_hi"][i] = prof.summary_len_range.low, prof.summary_len_range.high
        cols["conf"][i] = prof.confidence
        cols["qlen"][i] = rng.randint(*lp.input_range)
    w = dict(cols, chunk_size=np.int64(c["chunk"]), out_budget=np.int64(lp.out_budget),
             fixed_space=np.array([7, 1, 35, 30, 200] if c.get("full_space") else [0, 0, 0, 0, 0], dtype=np.int32))
    batch = refpath.Batch(rs, w)
    spaces, fb = batch.gate()
    per_tok = Mem.bytes_per_kv_token(batch.model)
    for i in range(n):
        if c.get("full_space"):
            cols["free"][i] = 16 * GiB - rng.randint(0, 16 * GiB)
        else:
            q = batch.queries[i]
            top = max(Mem.plan_bytes(q.query_token_len, cfg, c["chunk"], per_tok, lp.out_budget)
                      for cfg in M.enumerate_candidates(batch.spaces[i]))
            cols["free"][i] = rng.randint(0, 2 * top)
    batch.free = [int(x) for x in cols["free"]]
    w["free"] = cols["free"]
    pool = refpath.PoolSelect(batch, os.cpu_count())
    t0 = time.perf_counter()
    sel = pool.run()
    pool.close()
    print(f"{name}: {n} queries, select {time.perf_counter() - t0:.1f} s, gate fallbacks {int(fb.sum())}, "
          f"status counts {np.bincount(sel[:, 3], minlength=3).tolist()}")
    return dict(w, exp_space=spaces.astype(np.uint16), exp_gate_fb=fb, exp_select=sel)


def main():
    rs = refpath.import_ragsched(refpath.REF_SRC)
    for name in (sys.argv[1:] or CFGS):
        out = make(name, rs)
        np.savez_compressed(os.path.join(HERE, f"workload_{name}.npz"), **out)


if __name__ == "__main__":
    main()
