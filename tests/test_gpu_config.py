"""GPU parity of the config path (gate/prune, best-fit/fallback select,
KV-memory and delay models) against the reference's golden vectors and the
C oracle.  Bit-exact: these are integer / IEEE-double computations."""

import numpy as np
import pytest
import torch

from oracle import c_oracle
from oracle import config_oracle as co
from paper_2412_10543_b200 import _lib, batch
from tests import golden_data as gd

pytestmark = pytest.mark.gpu


def dev():
    return torch.device("cuda", 0)


def select_dev(spaces5, joint, qlen, free, p: co.SelectParams, allow_fallback=True, cost=None, running=None):
    n = len(qlen)
    sp = batch.spaces_from_arrays(*(np.asarray(spaces5)[:, i] for i in range(5)))
    prof = np.zeros(n, dtype=_lib.PROFILE_DTYPE)
    prof["needs_joint_reasoning"] = np.asarray(joint, dtype=np.uint8)
    params = batch.SelectParams(p.per_token_bytes, p.chunk_size, p.out_budget, p.template_tokens, p.max_chunks,
                                p.chunk_step, p.interlen_step, allow_fallback)
    out, delay = batch.select(batch.to_device(sp, dev()), batch.to_device(prof, dev()),
                              torch.as_tensor(np.asarray(qlen, dtype=np.int32), device=dev()),
                              torch.as_tensor(np.asarray(free, dtype=np.int64), device=dev()), params, cost=cost,
                              running_before=None if running is None else
                              torch.as_tensor(np.asarray(running, dtype=np.int32), device=dev()))
    cfg = batch.from_device(out, _lib.CONFIG_DTYPE)
    return cfg, (delay.cpu().numpy() if delay is not None else None)


def test_select_golden_bit_exact():
    psets = [co.SelectParams(**p) for p in gd.param_sets()]
    rows = gd.select_rows()
    for ps in range(len(psets)):
        sub = rows[rows[:, 0] == ps]
        cfg, _ = select_dev(sub[:, 1:6], sub[:, 6], sub[:, 7], sub[:, 8], psets[ps])
        np.testing.assert_array_equal(cfg["method"], sub[:, 9])
        np.testing.assert_array_equal(cfg["num_chunks"], sub[:, 10])
        np.testing.assert_array_equal(cfg["interlen"], sub[:, 11])
        np.testing.assert_array_equal(cfg["kv_bytes"], sub[:, 12])
        np.testing.assert_array_equal(cfg["status"], sub[:, 13])


def random_select_batch(rng, n, p, full_space_frac=0.3):
    m = rng.integers(1, 8, n)
    full = rng.random(n) < full_space_frac
    m[full] = 7
    lo = rng.integers(1, p.max_chunks + 1, n)
    hi = np.minimum(lo + rng.integers(0, p.max_chunks, n), p.max_chunks)
    lo[full], hi[full] = 1, p.max_chunks
    a = rng.integers(30, 201, n)
    b = np.minimum(a + rng.integers(0, 171, n), 200)
    a[full], b[full] = 30, 200
    a = np.where(m & 4, a, 0)
    b = np.where(m & 4, b, 0)
    spaces = np.stack([m, lo, hi, a, b], axis=1).astype(np.int32)
    joint = rng.integers(0, 2, n).astype(np.uint8)
    qlen = rng.integers(1, 12001, n).astype(np.int32)
    maxb = co.plan_bytes(12000, (4, p.max_chunks, 200), p) * 2
    free = np.where(rng.random(n) < 0.5, rng.integers(0, maxb, n), 16 * 1024**3 - rng.integers(0, 16 * 1024**3, n))
    return spaces, joint, qlen, free.astype(np.int64)


@pytest.mark.parametrize("pidx", range(8))
def test_select_random_vs_c_oracle(pidx):
    p = co.SelectParams(**gd.param_sets()[pidx])
    rng = np.random.default_rng(100 + pidx)
    spaces, joint, qlen, free = random_select_batch(rng, 20000, p)
    cfg, _ = select_dev(spaces, joint, qlen, free, p)
    ocfg, ob, ost = c_oracle.select_batch(spaces, joint, qlen, free, p)
    np.testing.assert_array_equal(cfg["status"], ost)
    np.testing.assert_array_equal(cfg["kv_bytes"], ob)
    np.testing.assert_array_equal(np.stack([cfg["method"], cfg["num_chunks"], cfg["interlen"]], 1), ocfg)


def test_select_cfg5_burst_full_space_100k():
    """cfg5: 100k queries x the full 700-candidate space, both free-memory regimes."""
    p = co.SelectParams(chunk_size=1000, out_budget=10)
    rng = np.random.default_rng(5)
    n = 100_000
    spaces = np.tile(np.array([[7, 1, 35, 30, 200]], dtype=np.int32), (n, 1))
    joint = rng.integers(0, 2, n).astype(np.uint8)
    qlen = rng.integers(400, 2001, n).astype(np.int32)
    maxb = co.plan_bytes(2000, (4, 35, 200), p)
    free = np.where(np.arange(n) % 2 == 0, rng.integers(0, 2 * maxb, n), 16 * 1024**3 - rng.integers(0, 16 * 1024**3, n))
    cfg, _ = select_dev(spaces, joint, qlen, free, p)
    ocfg, ob, ost = c_oracle.select_batch(spaces, joint, qlen, free, p)
    np.testing.assert_array_equal(cfg["status"], ost)
    np.testing.assert_array_equal(cfg["kv_bytes"], ob)
    np.testing.assert_array_equal(np.stack([cfg["method"], cfg["num_chunks"], cfg["interlen"]], 1), ocfg)
    # the full space holds map_rerank/1, the cheapest plan of all, so the
    # fallback can never beat it: only best-fit or MustQueue occur
    assert set(np.unique(ost).tolist()) == {0, 2}


def test_select_without_fallback_and_overflow_guard():
    p = co.SelectParams()
    spaces = np.array([[2, 5, 10, 0, 0], [2, 5, 10, 0, 0]], dtype=np.int32)
    cfg, _ = select_dev(spaces, [1, 1], [100, 100], [0, 10**15], p, allow_fallback=False)
    assert list(cfg["status"]) == [2, 0]
    huge = co.SelectParams(per_token_bytes=1 << 45)
    cfg, _ = select_dev(spaces[:1], [1], [100], [10**15], huge)
    assert cfg["status"][0] == _lib.RS_SELECT_OVERFLOW


def test_plan_delay_golden_bit_exact():
    z = gd.latency()
    psets = [co.SelectParams(**p) for p in gd.param_sets()]
    costs = z["costs"]
    for ci in range(len(costs)):
        for ps in range(len(psets)):
            sel = (z["plans"][:, 0] == ci) & (z["plans"][:, 1] == ps)
            if not sel.any():
                continue
            pl = z["plans"][sel]
            n = len(pl)
            # force the golden config through select: a singleton space with huge free memory
            spaces = np.stack([pl[:, 2], pl[:, 3], pl[:, 3], np.where(pl[:, 2] == 4, pl[:, 4], 0),
                               np.where(pl[:, 2] == 4, pl[:, 4], 0)], axis=1).astype(np.int32)
            cfg, delay = select_dev(spaces, np.zeros(n), pl[:, 5], np.full(n, 1 << 60), psets[ps],
                                    cost=batch.CostModel(*costs[ci]), running=pl[:, 6])
            assert (cfg["status"] == 0).all()
            np.testing.assert_array_equal(delay, z["plan_delay"][sel])  # bit-exact


def test_call_latency_golden_bit_exact():
    z = gd.latency()
    calls = z["calls"]
    for ci, c in enumerate(z["costs"]):
        sel = calls[:, 0] == ci
        t = lambda col: torch.as_tensor(calls[sel, col].astype(np.int64), device=dev())  # noqa: E731
        got = batch.call_latency_batch(t(1), t(2), t(3), batch.CostModel(*c)).cpu().numpy()
        np.testing.assert_array_equal(got, z["latency"][sel])


def test_plan_bytes_kernel_vs_oracle():
    rng = np.random.default_rng(9)
    for ps in gd.param_sets():
        p = co.SelectParams(**ps)
        n = 5000
        m = rng.choice([1, 2, 4], n).astype(np.uint8)
        nc = rng.integers(1, 36, n).astype(np.int32)
        il = rng.integers(1, 301, n).astype(np.int32)
        q = rng.integers(1, 12001, n).astype(np.int32)
        params = batch.SelectParams(p.per_token_bytes, p.chunk_size, p.out_budget, p.template_tokens)
        got = batch.plan_bytes_batch(*(torch.as_tensor(x, device=dev()) for x in (m, nc, il, q)), params).cpu().numpy()
        want = [co.plan_bytes(int(q[i]), (int(m[i]), int(nc[i]), int(il[i])), p) for i in range(n)]
        np.testing.assert_array_equal(got, want)


# -- gate ----------------------------------------------------------------------

def gate_dev(seq, chunk=None):
    n = len(seq["conf"])
    pr = seq["profiles"]
    prof = batch.profiles_from_arrays(pr[:, 0], pr[:, 1], pr[:, 2], pr[:, 3], pr[:, 4], seq["conf"])
    ds = seq["default_space"]
    window = batch.GateWindow(dev())
    if seq["prefill"]:
        rec = np.zeros(1, dtype=_lib.WINDOW_DTYPE)
        rec["spaces"][0, :len(seq["prefill"])] = batch.spaces_from_arrays(*np.array(seq["prefill"]).T)
        rec["len"] = len(seq["prefill"])
        window.tensor = batch.to_device(rec, dev()).reshape(-1)
    outs = []
    step = chunk or n
    for s in range(0, n, step):
        out = batch.prune_gate(batch.to_device(prof[s:s + step], dev()), window, threshold=seq["threshold"],
                               default_space=ds, max_chunks=seq["max_chunks"])
        outs.append(batch.from_device(out, _lib.SPACE_DTYPE))
    o = np.concatenate(outs)
    return np.stack([o["methods"], o["num_chunks_lo"], o["num_chunks_hi"], o["interlen_lo"], o["interlen_hi"],
                     o["gate_fallback"]], axis=1).astype(np.int32)


@pytest.mark.parametrize("seq", gd.gate_sequences(), ids=lambda s: s["name"])
def test_gate_golden_bit_exact(seq):
    np.testing.assert_array_equal(gate_dev(seq), seq["expected"])


@pytest.mark.parametrize("chunk", [1, 7, 1000, 1024, 1025])
def test_gate_window_carries_across_batches(chunk):
    seq = [s for s in gd.gate_sequences() if s["name"] == "heavy_noise"][0]
    np.testing.assert_array_equal(gate_dev(seq, chunk=chunk), seq["expected"])


def test_gate_large_batch_vs_c_oracle():
    rng = np.random.default_rng(3)
    n = 300_000
    prof = np.stack([rng.integers(0, 2, n), rng.integers(0, 2, n), rng.integers(1, 11, n),
                     rng.integers(30, 120, n), rng.integers(120, 201, n)], axis=1).astype(np.int32)
    conf = np.where(rng.random(n) < 0.2, rng.uniform(0.55, 0.88, n), 0.99)
    conf[1000:1400] = 0.5  # a long rejected run
    seq = dict(profiles=prof, conf=conf, threshold=0.9, default_space=(2, 1, 5, 0, 0), max_chunks=35, prefill=[])
    got = gate_dev(seq)
    out, fb, _ = c_oracle.gate_batch(prof, conf)
    np.testing.assert_array_equal(got, np.concatenate([out, fb[:, None]], axis=1))


def test_gate_rejects_bad_threshold():
    prof = batch.to_device(batch.profiles_from_arrays([1], [1], [3], [40], [50], [0.95]), dev())
    with pytest.raises(ValueError):
        batch.prune_gate(prof, batch.GateWindow(dev()), threshold=0.0)
    with pytest.raises(ValueError):
        batch.prune_gate(prof, batch.GateWindow(dev()), threshold=1.5)


def test_plan_calls_golden_bit_exact():
    """§8(f2): per-call expansion of chosen configs vs the reference's plan_calls."""
    psets = gd.param_sets()
    rows, calls = gd.plan_calls()
    want_calls = {}
    for c in calls:
        want_calls.setdefault(int(c[0]), []).append(tuple(int(x) for x in c[1:]))
    for ps in range(len(psets)):
        for max_ctx in np.unique(rows[:, 2]):
            sel = (rows[:, 1] == ps) & (rows[:, 2] == max_ctx)
            if not sel.any():
                continue
            sub = rows[sel]
            cfg = np.zeros(len(sub), dtype=_lib.CONFIG_DTYPE)
            cfg["method"], cfg["num_chunks"], cfg["interlen"] = sub[:, 3], sub[:, 4], sub[:, 5]
            cfg["status"] = 0
            p = psets[ps]
            params = batch.SelectParams(p["per_token_bytes"], p["chunk_size"], p["out_budget"], p["template_tokens"],
                                        p["max_chunks"])
            off, cl, tot, st = batch.plan_calls(batch.to_device(cfg, dev()),
                                                torch.as_tensor(sub[:, 6].astype(np.int32), device=dev()), params,
                                                int(max_ctx))
            off = off.cpu().numpy()
            cl = batch.from_device(cl, _lib.CALL_DTYPE) if off[-1] else np.zeros(0, dtype=_lib.CALL_DTYPE)
            st, tot = st.cpu().numpy(), tot.cpu().numpy()
            for j, r in enumerate(sub):
                trial, status, total = int(r[0]), int(r[7]), int(r[8])
                assert int(st[j]) == status, (trial, int(st[j]), status)
                seg = cl[off[j]:off[j + 1]]
                got = [(int(c["kind"]), int(c["prompt_tokens"]), int(c["max_output_tokens"]), int(c["kv_bytes"]),
                        int(c["index"])) for c in seg]
                assert got == want_calls.get(trial, []), trial
                if status == 0:
                    assert int(tot[j]) == total
