"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no TUF, no priority, no stop
rule, no paging, no model math).  It only produces inputs:

* vocabularies with a token -> (skill, E_min) table   (``vocab``)
* scripted robot plans shaped like the paper's traces  (``traces``)
* Poisson workload compositions (tab:data_sample)      (``workload``)
* model / engine configuration presets (BASELINE.json) (``configs``)

Every generator is deterministic given its seed (numpy PCG64).
"""
from .configs import ModelShape, EngineParams, MODEL_SHAPES, engine_params  # noqa: F401
from .vocab import SkillVocab, make_vocab  # noqa: F401
from .traces import Trace, make_trace, TRACE_CLASSES  # noqa: F401
from .workload import Request, compose_workload, closed_loop_requests  # noqa: F401
