"""Material parameters (pkg/src/vbdsim/materials.py:25-41).

The element arithmetic itself lives in the sm_100a kernel (csrc/vbd_common.cuh
``tet_contrib``): Stable Neo-Hookean Psi = mu/2 (I_C - 3) + lam/2 (J - gamma)^2,
gamma = 1 + mu/lam, with Rayleigh-style damping k_d.
"""

from dataclasses import dataclass


@dataclass(frozen=True)
class MaterialParams:
    mu: float
    lam: float
    k_d: float = 0.0

    def __post_init__(self):
        if self.mu <= 0.0:
            raise ValueError("mu must be positive")
        if self.lam <= 0.0:
            raise ValueError("lambda must be positive")
        if self.k_d < 0.0:
            raise ValueError("k_d must be >= 0")

    @property
    def gamma(self) -> float:
        return 1.0 + self.mu / self.lam
