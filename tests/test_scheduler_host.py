"""CPU check of the Scheduler mirror's host logic (backlog, per-call state,
completions, trace, exception mapping) and of the oracle's restatement of the
admission chain: the reference Scheduler traces (tests/golden/
make_sched_golden.py, incl. the runs recorded inside sim.run) are replayed
with the GPU entry points (rs_admit_fifo, rs_plan_calls) swapped — in this
test only — for oracle/config_oracle.admit_chain / plan_calls that fill the
same C-struct byte layouts.  The GPU replay of the same traces is
tests/test_gpu_scheduler.py."""

import numpy as np
import pytest
import torch

from oracle import config_oracle as co
from paper_2412_10543_b200 import _lib
from paper_2412_10543_b200 import scheduler as S
from tests import test_gpu_scheduler as T

_STOP = {co.ADMIT_DRAINED: _lib.RS_ADMIT_DRAINED, co.ADMIT_BLOCKED: _lib.RS_ADMIT_BLOCKED,
         co.ADMIT_NO_PROFILE: _lib.RS_ADMIT_NO_PROFILE, co.ADMIT_IMPOSSIBLE: _lib.RS_ADMIT_IMPOSSIBLE,
         co.ADMIT_FIXED_SPACE: _lib.RS_ADMIT_FIXED_SPACE, co.ADMIT_INVALID_CHUNKS: _lib.RS_ADMIT_INVALID_CHUNKS,
         co.ADMIT_CONTEXT_OVERFLOW: _lib.RS_ADMIT_CONTEXT_OVERFLOW, co.ADMIT_BAD_INTERLEN: _lib.RS_ADMIT_BAD_INTERLEN}


def _oparams(p):
    return co.SelectParams(p.per_token_bytes, p.chunk_size, p.out_budget, p.template_tokens, p.max_chunks,
                           p.chunk_step, p.interlen_step)


def _to_u8(rec):
    return torch.from_numpy(np.ascontiguousarray(rec).view(np.uint8).reshape(len(rec), rec.dtype.itemsize).copy())


def fake_admit_fifo(spaces, profiles, qlen, params, *, capacity_bytes, used_bytes, max_context_tokens,
                    has_profile=None, stream=None):
    n = spaces.shape[0]
    sp = spaces.numpy().reshape(-1).view(_lib.SPACE_DTYPE)
    pr = profiles.numpy().reshape(-1).view(_lib.PROFILE_DTYPE)
    hp = has_profile.numpy() if has_profile is not None else np.ones(n, np.uint8)
    ql = qlen.numpy()
    entries = [((int(s["methods"]), int(s["num_chunks_lo"]), int(s["num_chunks_hi"]), int(s["interlen_lo"]),
                 int(s["interlen_hi"])), bool(p["needs_joint_reasoning"]), bool(h), int(q))
               for s, p, h, q in zip(sp, pr, hp, ql)]
    adm, used, stop, stop_cfg = co.admit_chain(entries, _oparams(params), capacity_bytes, used_bytes,
                                               max_context_tokens, params.allow_fallback)
    cfg = np.zeros(max(n, 1), _lib.CONFIG_DTYPE)
    info = np.zeros(max(n, 1), _lib.ADMIT_INFO_DTYPE)
    for i, ((m, nc, il), b, st, ab, na, fixed) in enumerate(adm):
        cfg[i] = (b, m, st, nc, il, 0)
        info[i] = (ab, na, int(fixed))
    if stop_cfg is not None:
        m, nc, il = stop_cfg
        cfg[len(adm)] = (0, m, 0, nc, il, 0)
    res = np.zeros(1, _lib.ADMIT_RESULT_DTYPE)
    res[0] = (n if stop == co.ADMIT_DRAINED else len(adm), used, _STOP[stop], 0)
    return _to_u8(cfg)[:n], _to_u8(info)[:n], _to_u8(res).reshape(-1)


def fake_plan_calls(configs, qlen, params, max_context_tokens, stream=None):
    c = configs.numpy().reshape(-1).view(_lib.CONFIG_DTYPE)
    ql = qlen.numpy()
    p = _oparams(params)
    offs, recs, totals, status = [0], [], [], []
    for r, q in zip(c, ql):
        st, calls, total = co.plan_calls(int(q), (int(r["method"]), int(r["num_chunks"]), int(r["interlen"])), p,
                                         max_context_tokens)
        for kind, prompt, out, kv, idx in calls:
            recs.append((kv, prompt, out, idx, kind, 0, 0))
        offs.append(offs[-1] + len(calls))
        totals.append(total)
        status.append(st)
    calls = np.array(recs, dtype=_lib.CALL_DTYPE) if recs else np.zeros(0, _lib.CALL_DTYPE)
    return (torch.tensor(offs, dtype=torch.int64), _to_u8(calls) if len(calls) else torch.zeros((0, 24), torch.uint8),
            torch.tensor(totals, dtype=torch.int64), torch.tensor(status, dtype=torch.uint8))


class FakeArena:
    """scalar.AdmitArena's interface over host numpy arrays, filled by the
    oracle's restatement of the two kernels instead of the GPU."""

    def __init__(self):
        self.cap = 0
        self.ensure(32)

    def ensure(self, n):
        if n <= self.cap:
            return
        self.cap = max(n, 2 * self.cap)
        self.spaces = np.zeros((self.cap, 16), np.uint8)
        self.profiles = np.zeros((self.cap, 16), np.uint8)
        self.hasprof = np.zeros(self.cap, np.uint8)
        self.qlen = np.zeros(self.cap, np.int32)
        self.configs = np.zeros(self.cap, _lib.CONFIG_DTYPE)
        self.info = np.zeros(self.cap, _lib.ADMIT_INFO_DTYPE)

    def admit(self, n, params_c, capacity, used, max_ctx):
        p = self._params(params_c)
        cfg, info, res = fake_admit_fifo(torch.from_numpy(self.spaces[:n]), torch.from_numpy(self.profiles[:n]),
                                         torch.from_numpy(self.qlen[:n]), p, capacity_bytes=capacity,
                                         used_bytes=used, max_context_tokens=max_ctx,
                                         has_profile=torch.from_numpy(self.hasprof[:n]))
        self.configs[:n] = cfg.numpy().reshape(-1).view(_lib.CONFIG_DTYPE)
        self.info[:n] = info.numpy().reshape(-1).view(_lib.ADMIT_INFO_DTYPE)
        r = res.numpy().view(_lib.ADMIT_RESULT_DTYPE)[0]
        return int(r["admitted"]), int(r["stop"])

    def admit_and_plan(self, n, params_c, capacity, used, max_ctx):
        # the GPU arena runs the plan expansion over all n entries in stream
        # order; the restated chain plans the admitted prefix (what the
        # scheduler reads)
        m, stop = self.admit(n, params_c, capacity, used, max_ctx)
        return m, stop, (self.plan_calls(m, params_c, max_ctx) if m else None)

    def plan_calls(self, m, params_c, max_ctx):
        cfg = torch.from_numpy(self.configs[:m].view(np.uint8).reshape(m, 16))
        off, calls, tot, st = fake_plan_calls(cfg, torch.from_numpy(self.qlen[:m]), self._params(params_c), max_ctx)
        rec = calls.numpy().reshape(-1).view(_lib.CALL_DTYPE) if calls.numel() else np.zeros(0, _lib.CALL_DTYPE)
        return off.numpy(), rec, tot.numpy(), st.numpy()

    @staticmethod
    def _params(c):
        from paper_2412_10543_b200 import batch

        return batch.SelectParams(c.per_token_bytes, c.chunk_size, c.out_budget, c.template_tokens, c.max_chunks,
                                  c.chunk_step, c.interlen_step, bool(c.allow_fallback))


@pytest.fixture()
def oracle_backed(monkeypatch):
    monkeypatch.setattr(S.Scheduler, "_arena", lambda self: self.__dict__.setdefault("_fake_arena", FakeArena()))


@pytest.mark.parametrize("rec", T.TRACES, ids=[r["name"] for r in T.TRACES])
def test_scheduler_host_logic_replays_reference(rec, oracle_backed):
    T.test_scheduler_replays_reference_trace(rec)
