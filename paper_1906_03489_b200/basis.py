"""Basis keys (mirror of spechp.basis, basis.py:26-53)."""
from __future__ import annotations

import warnings
from dataclasses import dataclass
from enum import Enum

from .quadrature import PointsKey


class BasisType(Enum):
    MODIFIED_A = "modified_a"
    MODIFIED_B = "modified_b"
    LAGRANGE_GLL = "lagrange_gll"


class BasisError(ValueError):
    pass


@dataclass(frozen=True)
class BasisKey:
    basis_type: BasisType
    num_modes: int
    points_key: PointsKey

    def __post_init__(self):
        if not isinstance(self.num_modes, int) or self.num_modes < 1:
            raise BasisError(f"num_modes must be positive, got {self.num_modes!r}")
        if self.basis_type is BasisType.MODIFIED_A and self.num_modes < 2:
            raise BasisError("modified basis needs num_modes >= 2 "
                             "(both boundary modes are always present)")
        if self.points_key.num_points < self.num_modes:
            warnings.warn(
                f"quadrature count {self.points_key.num_points} below mode "
                f"count {self.num_modes}; transforms will be rank-deficient",
                stacklevel=2)

    @property
    def order(self):
        return self.num_modes - 1
