"""B200-native (sm_100a) implementation of Aragog's two data-parallel hot
paths (arXiv 2511.20975): routing (enumerate / chain modes) and per-stage
just-in-time scheduling, behind the C ABI in include/aragog_b200.h."""
from ._capi import AgError, ValidationError, lib  # noqa: F401
from .routing import (AccuracyBatch, ConfigSpace, Device, DeviceAccuracyBatch,  # noqa: F401
                      GenParams, NoisyRouter, OracleRouter, RouteResult, enumerate_members)
from .predictor import ConfigPredictor, PredictionBatch  # noqa: F401,E402
from .scheduler import (PER_INPUT_RUNTIME_COST, PER_INPUT_STATIC, Assignment, Engines, Queue, audit_round_fairness,  # noqa: F401,E402
                        RuntimeCostContext, SchedSession, beam_schedule, select_bitmap, select_bitmap_stats,
                        select_per_input, select_per_input_host, select_per_workflow)
