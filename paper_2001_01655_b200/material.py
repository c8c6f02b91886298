"""SIMP law (mirrors reference material.py:8-50); ``modulus`` on CUDA tensors
runs on the device through the C-ABI, numpy inputs stay numpy."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._dev import empty_dev, ptr, stream_ptr


@dataclass(frozen=True)
class SimpLaw:
    e_max: float = 1.0
    penalty: float = 3.0
    e_min_ratio: float = 1e-10

    @property
    def e_min(self):
        return self.e_min_ratio * self.e_max

    def modulus(self, rho):
        if hasattr(rho, "is_cuda") and rho.is_cuda:
            out = empty_dev(rho.numel())
            _lib.check(_lib.load().tmg_simp_modulus(ptr(rho.contiguous()), rho.numel(), float(self.penalty),
                                                    float(self.e_max), float(self.e_min), ptr(out),
                                                    stream_ptr(None)))
            return out
        rho = np.asarray(rho, dtype=float)
        if np.any((rho < 0) | (rho > 1)):
            raise ValueError("rho must lie in [0, 1]")
        return self.e_min + (self.e_max - self.e_min) * rho ** self.penalty

    def modulus_derivative(self, rho):
        rho = np.asarray(rho, dtype=float)
        p = self.penalty
        if p == 1.0:
            return np.full_like(rho, self.e_max - self.e_min)
        return p * (self.e_max - self.e_min) * rho ** (p - 1.0)
