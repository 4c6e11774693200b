"""Parity taps for include/satgrad/autodiff.hpp, run on the device.

``forward`` / ``backward`` execute the same sm_100a kernels the sampler uses,
over every node of the circuit (not just the output cone), and return the
reference's layouts: tape ``[n_nodes][batch]`` in reference node order,
``y`` / ``dv`` / ``dp`` row-major ``[batch][cols]``.  ``input_cols`` must be
the circuit's constrained-PI order (the V column order of run()).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .sampler import DeviceCircuit, device_context


def embed(v, device: int = 0) -> np.ndarray:
    """autodiff.cpp:57-62 (bit-exact clamped sigmoid)."""
    v = np.ascontiguousarray(v, np.float32)
    out = np.zeros_like(v)
    if v.size:
        _lib.check(_lib.load().sgx_embed(device_context(device), _lib.ptr(v, C.c_float), v.size,
                                         _lib.ptr(out, C.c_float)))
    return out


def expf(x, device: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    out = np.zeros_like(x)
    if x.size:
        _lib.check(_lib.load().sgx_expf(device_context(device), _lib.ptr(x, C.c_float), x.size,
                                        _lib.ptr(out, C.c_float)))
    return out


def forward(dc: DeviceCircuit, p) -> tuple[np.ndarray, np.ndarray]:
    """autodiff.cpp:64-152."""
    p = np.ascontiguousarray(p, np.float32)
    batch = p.shape[0]
    n, m = dc.circuit.n_nodes, len(dc.circuit.out_var)
    tape = np.zeros((n, batch), np.float32)
    y = np.zeros((batch, m), np.float32)
    _lib.check(_lib.load().sgx_forward(dc.h, _lib.ptr(p, C.c_float) if p.size else None, batch,
                                       _lib.ptr(tape, C.c_float), _lib.ptr(y, C.c_float)))
    return tape, y


def backward(dc: DeviceCircuit, tape, v) -> tuple[np.ndarray, np.ndarray]:
    """autodiff.cpp:172-283 with the circuit's output targets."""
    tape = np.ascontiguousarray(tape, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    batch = tape.shape[1]
    dv = np.zeros(v.shape, np.float32)
    dp = np.zeros(v.shape, np.float32)
    _lib.check(_lib.load().sgx_backward(dc.h, _lib.ptr(tape, C.c_float), batch,
                                        _lib.ptr(v, C.c_float) if v.size else None,
                                        _lib.ptr(dv, C.c_float) if v.size else None,
                                        _lib.ptr(dp, C.c_float) if v.size else None))
    return dv, dp
