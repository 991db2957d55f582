"""Install the GPU hot path into the reference package ``ragsched``.

The reference resolves its hot-path functions by module attribute
(``Scheduler._try_admit_new`` calls ``best_fit_select`` / ``fallback_config``
from ``ragsched.scheduler``, scheduler.py:340/:360; ``QueryProfiler.gate``
calls ``gate_profile`` from ``ragsched.profiler``, profiler.py:534-541).
``install(ragsched)`` rebinds those names to wrappers that run this package's
kernels and return the reference's own classes (``RagConfig``,
``PrunedConfigSpace``, ``GateDecision``), so dataclass equality and the rest
of the reference pipeline are unchanged.
"""

from __future__ import annotations

import functools
from types import SimpleNamespace

from . import mapping as _mapping
from . import memory as _memory
from . import profiler as _profiler
from . import scheduler as _scheduler
from . import sim as _sim


def scheduler_class(ragsched_pkg):
    """This package's GPU-backed Scheduler (FIFO admission chain on the
    device, scheduler.py:194-469) building the reference's own Admission /
    AdmittedCall / CompletionInfo / QueryRun / CallPlan objects and raising
    its own exceptions."""
    import importlib

    sched = importlib.import_module(ragsched_pkg.__name__ + ".scheduler")
    memory = importlib.import_module(ragsched_pkg.__name__ + ".memory")
    types = importlib.import_module(ragsched_pkg.__name__ + ".types")
    ns = SimpleNamespace(
        Admission=sched.Admission, AdmittedCall=sched.AdmittedCall, CompletionInfo=sched.CompletionInfo,
        QueryRun=sched.QueryRun, UnknownCall=sched.UnknownCall, MemorySafetyViolation=sched.MemorySafetyViolation,
        SchedulingImpossible=sched.SchedulingImpossible, InvalidChunkCount=types.InvalidChunkCount,
        ContextOverflow=types.ContextOverflow, RagConfig=types.RagConfig, SynthesisMethod=types.SynthesisMethod,
        LlmCall=memory.LlmCall, CallPlan=memory.CallPlan, CallKind=memory.CallKind)
    return type("Scheduler", (_scheduler.Scheduler,), {"classes": ns, "__module__": __name__})


def install(ragsched_pkg) -> dict:
    """Patch ``ragsched.{scheduler,profiler,mapping,memory,sim}``.  Returns the
    originals (for ``uninstall``)."""
    import importlib

    sched = importlib.import_module(ragsched_pkg.__name__ + ".scheduler")
    prof = importlib.import_module(ragsched_pkg.__name__ + ".profiler")
    mapping = importlib.import_module(ragsched_pkg.__name__ + ".mapping")
    memory = importlib.import_module(ragsched_pkg.__name__ + ".memory")
    sim = importlib.import_module(ragsched_pkg.__name__ + ".sim")
    types = importlib.import_module(ragsched_pkg.__name__ + ".types")
    kw_cfg = dict(config_cls=types.RagConfig, method_enum=types.SynthesisMethod)
    kw_space = dict(space_cls=mapping.PrunedConfigSpace, method_enum=types.SynthesisMethod,
                    range_cls=types.IntRange)

    originals = {
        (sched, "best_fit_select"): sched.best_fit_select,
        (sched, "fallback_config"): sched.fallback_config,
        (prof, "gate_profile"): prof.gate_profile,
        (prof, "map_profile"): prof.map_profile,
        (mapping, "map_profile"): mapping.map_profile,
        (memory, "plan_bytes"): memory.plan_bytes,
        (sim, "call_latency"): sim.call_latency,
        (sched, "Scheduler"): sched.Scheduler,
        (sim, "Scheduler"): sim.Scheduler,
        (memory, "plan_calls"): memory.plan_calls,
        (prof, "parse_profile_text"): prof.parse_profile_text,
        (sched, "plan_calls"): sched.plan_calls,
        (prof, "_per_field_confidences"): prof._per_field_confidences,
    }

    sched.best_fit_select = functools.partial(_scheduler.best_fit_select, **kw_cfg)
    sched.fallback_config = functools.partial(_scheduler.fallback_config, **kw_cfg)
    prof.gate_profile = functools.partial(_profiler.gate_profile, decision_cls=prof.GateDecision,
                                          default_space=prof.DEFAULT_FALLBACK_SPACE, **kw_space)
    mp = functools.partial(_mapping.map_profile, **kw_space)
    prof.map_profile = mp
    mapping.map_profile = mp
    memory.plan_bytes = _memory.plan_bytes
    sim.call_latency = _sim.call_latency
    gpu_sched = scheduler_class(ragsched_pkg)
    sched.Scheduler = gpu_sched
    sim.Scheduler = gpu_sched
    pc = functools.partial(_memory.plan_calls, call_cls=memory.LlmCall, plan_cls=memory.CallPlan,
                           kind_enum=memory.CallKind)
    memory.plan_calls = pc
    sched.plan_calls = pc
    prof.parse_profile_text = functools.partial(_profiler.parse_profile_text, profile_cls=mapping.QueryProfile,
                                                range_cls=types.IntRange, exc_cls=prof.UnparseableAnswer)
    prof._per_field_confidences = _profiler.per_field_confidences
    return originals


def uninstall(originals: dict) -> None:
    for (mod, name), fn in originals.items():
        setattr(mod, name, fn)
