"""Chain-mode routing: host mirror of ConfigPredictor over the C ABI.

Reference: include/aragog/predictor.h:70-103, src/predictor.cpp:107-262.
The chain plan is built once per space on the host; predict() for a whole
batch of requests runs in one kernel (one warp per request).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import check, lib
from .routing import Device, DeviceAccuracyBatch, _ptr

INF = math.inf


class PredictOut(C.Structure):
    _fields_ = [("viable", C.c_void_p), ("viable_stride", C.c_int32), ("n_viable", C.c_void_p),
                ("search_evals", C.c_void_p), ("verify_evals", C.c_void_p),
                ("router_time", C.c_void_p), ("truncated", C.c_void_p)]


@dataclass
class PredictionBatch:
    """PredictionResult (predictor.h:75-83) for every request of a batch."""
    viable: object        # [R, stride] int32 tensor (canonical indices)
    n_viable: object      # [R]
    search_evals: object  # [R]
    verify_evals: object  # [R]
    router_time: object   # [R] float64
    truncated: object     # [R] uint8

    def viable_of(self, r):
        return self.viable[r, : int(self.n_viable[r])]


class ConfigPredictor:
    """ConfigPredictor(space, router, PredictorParams{chain_cap, exhaustive_limit})."""

    def __init__(self, device: Device, chain_cap: int = 0, exhaustive_limit: int = 4096):
        self.device = device
        h = C.c_void_p()
        check(lib().ag_predictor_create(device.handle, chain_cap, C.c_uint64(exhaustive_limit),
                                        C.byref(h)))
        self._h = h
        nc, ln, ex, nu = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        check(lib().ag_predictor_info(h, C.byref(nc), C.byref(ln), C.byref(ex), C.byref(nu), None))
        self.n_chains, self.chain_len, self.n_unique = nc.value, ln.value, nu.value
        self.exhaustive = bool(ex.value)

    def chains(self) -> np.ndarray:
        """ChainPlan::chains as canonical indices [n_chains, chain_len]."""
        out = np.zeros(self.n_chains * self.chain_len, np.uint64)
        check(lib().ag_predictor_info(self._h, None, None, None, None, C.c_void_p(_ptr(out))))
        return out.reshape(self.n_chains, self.chain_len)

    def predict_batch(self, truth: DeviceAccuracyBatch, router, budget=INF) -> PredictionBatch:
        """predict(request_ids[r], budget[r]) for every row (async on the ctx stream).
        `budget` is a scalar or a device float64 tensor [R]."""
        import torch

        R = truth.n_requests
        dev = self.device.torch_device
        stride = max(1, self.n_unique)
        res = PredictionBatch(
            viable=torch.zeros((R, stride), dtype=torch.int32, device=dev),
            n_viable=torch.zeros(R, dtype=torch.int32, device=dev),
            search_evals=torch.zeros(R, dtype=torch.int32, device=dev),
            verify_evals=torch.zeros(R, dtype=torch.int32, device=dev),
            router_time=torch.zeros(R, dtype=torch.float64, device=dev),
            truncated=torch.zeros(R, dtype=torch.uint8, device=dev))
        out = PredictOut(_ptr(res.viable), stride, _ptr(res.n_viable), _ptr(res.search_evals),
                         _ptr(res.verify_evals), _ptr(res.router_time), _ptr(res.truncated))
        if isinstance(budget, (int, float)):
            bptr, ball = None, float(budget)
        else:
            bptr, ball = _ptr(budget), 0.0
        t = truth.c_struct()
        check(lib().ag_predict(self._h, C.byref(t), C.byref(router), C.c_void_p(bptr),
                               C.c_double(ball), C.byref(out)))
        return res

    def __del__(self):
        try:  # module globals may already be gone at interpreter shutdown
            _capi.release("ag_predictor_destroy", getattr(self, "_h", None))
        except Exception:  # noqa: BLE001
            pass
        self._h = None
