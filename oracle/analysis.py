"""Appendix B closed form -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:596-610: for independent w1 ~ N(0, s1^2), w2 ~ N(0, s2^2),
  P(| |w1|-|w2| | / (|w1|+|w2|) < tau) =
      (2/pi) [ atan(rho (1+tau)/(1-tau)) - atan(rho (1-tau)/(1+tau)) ],  rho = s2/s1.
"""
from __future__ import annotations

import math


def similarity_fraction_closed(sigma_ratio: float, tau: float) -> float:
    if not (sigma_ratio > 0.0) or not (0.0 <= tau < 1.0):
        raise ValueError("DomainError: need sigma_ratio > 0 and 0 <= tau < 1")
    a = (1.0 - tau) / (1.0 + tau)
    b = (1.0 + tau) / (1.0 - tau)
    return (2.0 / math.pi) * (math.atan(sigma_ratio * b) - math.atan(sigma_ratio * a))
