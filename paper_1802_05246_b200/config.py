"""Scheme and boundary configuration (drop-in for hermwave's SchemeConfig,
BoundarySpec, BoundarySpec2D).

Semantics follow pkg/src/hermwave/dissipative.py:40-74 and
pkg/src/hermwave/boundary.py:24-53: same fields, defaults, validation and
messages.  Reflection itself never happens on the host — the kernels fold
the ghost signs into their loads (csrc/common.cuh).
"""

from __future__ import annotations

from dataclasses import dataclass, field

KINDS = ("periodic", "dirichlet0", "neumann0")


@dataclass(frozen=True)
class SchemeConfig:
    """m: method order; speed: wave speed c; lam: CFL number c*dt/h (min h in
    2D); stage_cap: optional Taylor stage cap (default 2m in 1D, 4m+4 in 2D)."""

    m: int
    speed: float = 1.0
    lam: float = 0.8
    stage_cap: int | None = None

    def __post_init__(self):
        if self.m < 1:
            raise ValueError(f"method order must be >= 1, got {self.m}")
        if not (0.0 < self.lam <= 1.0):
            raise ValueError(f"CFL number must be in (0, 1], got {self.lam}")
        if self.speed <= 0.0:
            raise ValueError("wave speed must be positive")
        if self.stage_cap is not None and self.stage_cap < 1:
            raise ValueError("stage cap must be at least 1")

    def dt(self, h: float) -> float:
        return self.lam * h / self.speed

    def stages_1d(self) -> int:
        return self.stage_cap if self.stage_cap is not None else 2 * self.m

    def stages_2d(self) -> int:
        return self.stage_cap if self.stage_cap is not None else 4 * self.m + 4


@dataclass(frozen=True)
class BoundarySpec:
    """Per-axis edge conditions; values are constant Dirichlet data."""

    left: str = "periodic"
    right: str = "periodic"
    left_value: float = 0.0
    right_value: float = 0.0

    def __post_init__(self):
        for side in (self.left, self.right):
            if side not in KINDS:
                raise ValueError(f"unknown boundary kind {side!r}, expected one of {KINDS}")
        if (self.left == "periodic") ^ (self.right == "periodic"):
            raise ValueError("periodic must be specified on both opposing sides")

    @property
    def periodic(self) -> bool:
        return self.left == "periodic"


@dataclass(frozen=True)
class BoundarySpec2D:
    x: BoundarySpec = field(default_factory=BoundarySpec)
    y: BoundarySpec = field(default_factory=BoundarySpec)


def check_periodicity(spec: BoundarySpec, grid_periodic: bool) -> None:
    # boundary.py:142-143,157-159
    if spec.periodic != grid_periodic:
        raise ValueError("boundary spec and grid disagree about periodicity")
