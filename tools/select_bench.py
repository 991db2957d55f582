"""Throughput of the config path kernels alone (cfg5: 100k queries x the full
700-candidate space, best-fit against varying free KV memory)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10543_b200 import batch  # noqa: E402


def main(n=100_000, reps=50):
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    sp = batch.spaces_from_arrays(np.full(n, 7), np.full(n, 1), np.full(n, 35), np.full(n, 30), np.full(n, 200))
    prof = batch.profiles_from_arrays(rng.integers(0, 2, n), rng.integers(0, 2, n), rng.integers(1, 11, n),
                                      np.full(n, 30), np.full(n, 200), np.where(rng.random(n) < 0.05, 0.6, 0.99))
    spaces, profiles = batch.to_device(sp, dev), batch.to_device(prof, dev)
    qlen = torch.as_tensor(rng.integers(400, 2001, n).astype(np.int32), device=dev)
    free = torch.as_tensor((16 * 1024**3 - rng.integers(0, 16 * 1024**3, n)).astype(np.int64), device=dev)
    params = batch.SelectParams(per_token_bytes=131072, chunk_size=1000, out_budget=10)
    cost = batch.CostModel()
    window = batch.GateWindow(dev)
    out = torch.empty((n, 16), dtype=torch.uint8, device=dev)
    # the full cost table (every candidate's bytes + plan delay): 70M records
    for _ in range(2):
        off, recs = batch.candidate_costs(spaces, qlen, params, cost=cost)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps_t = 5
    for _ in range(reps_t):
        off, recs = batch.candidate_costs(spaces, qlen, params, cost=cost)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps_t
    print(f"{'cost table (2 passes)':22s} {ms * 1e3:8.1f} us/batch  {n / ms * 1e3 / 1e6:8.1f} M queries/s  "
          f"{recs.shape[0] / ms * 1e3 / 1e9:8.2f} G candidates/s  ({recs.numel() / ms * 1e3 / 1e9:.0f} GB/s written)")
    del off, recs
    for mode in ("select", "select+delay", "gate", "gate+select+delay"):
        def step():
            if "gate" in mode:
                batch.prune_gate(profiles, window)
            if "select" in mode:
                batch.select(spaces, profiles, qlen, free, params, cost=cost if "delay" in mode else None, out=out)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        evals = n * 700 if "select" in mode else 0
        print(f"{mode:22s} {ms * 1e3:8.1f} us/batch  {n / ms * 1e3 / 1e6:8.1f} M queries/s  "
              f"{evals / ms * 1e3 / 1e9:8.2f} G candidate-evals/s")


if __name__ == "__main__":
    main()
