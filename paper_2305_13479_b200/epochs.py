"""Epoch arithmetic in exact rationals (reference pkg/src/collsched/epochs.py).

The LP's capacities and link delays are computed here on the host, in the
same snapped-rational arithmetic as the reference (epochs.py:107-123), so the
device builder receives bit-identical float64 capacities and integer delays.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from .errors import ValidationError

SLOWEST = "slowest"
FASTEST = "fastest"


@dataclass(frozen=True)
class EpochConfig:
    tau: float  # seconds per epoch
    K: int  # epochs 0..K-1
    duration_mode: str = SLOWEST
    epoch_multiplier: int = 1
    chunk_size: int = 1  # bytes

    def __post_init__(self):
        if self.tau <= 0:
            raise ValidationError("tau must be positive")
        if self.K < 1:
            raise ValidationError("K must be >= 1")
        if self.epoch_multiplier < 1:
            raise ValidationError("epoch_multiplier must be >= 1")
        if self.duration_mode not in (SLOWEST, FASTEST):
            raise ValidationError(f"unknown duration mode {self.duration_mode!r}")

    def with_horizon(self, K: int) -> "EpochConfig":
        return EpochConfig(self.tau, K, self.duration_mode, self.epoch_multiplier, self.chunk_size)


def snap(x) -> Fraction:
    """Nearest short rational, so 5e-7 s or 25e9 B/s divide exactly."""
    if isinstance(x, Fraction):
        return x
    if isinstance(x, int):
        return Fraction(x)
    return Fraction(x).limit_denominator(10 ** 12)


def ceil_q(q: Fraction) -> int:
    return -int((-q) // 1) if q > 0 else 0


def epoch_duration(t, chunk_size: int, mode: str = FASTEST, em: int = 1) -> float:
    caps = [e.capacity for e in t.edges]
    if not caps:
        raise ValidationError("topology has no edges")
    ref = min(caps) if mode == SLOWEST else max(caps)
    return float(em * Fraction(chunk_size) / snap(ref))


def compute_delta(edge, tau: float) -> int:
    """ceil(alpha / tau) epochs; 0 for a zero-latency link."""
    if tau <= 0:
        raise ValidationError("tau must be positive")
    if edge.alpha == 0:
        return 0
    return ceil_q(snap(edge.alpha) / snap(tau))


def cap_chunks(t, edge, k: int, cfg: EpochConfig) -> Fraction:
    """Chunks per epoch the edge carries during epoch k."""
    return snap(t.capacity_at(edge, k)) * snap(cfg.tau) / Fraction(cfg.chunk_size)
