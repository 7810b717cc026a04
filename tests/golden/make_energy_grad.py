"""Golden fixture for density_energy_and_gradient from the
REFERENCE implementation itself (run in the build container):

    python tests/golden/make_energy_grad.py

Writes energy_grad.npz: two charge clouds (a random 16x12x8 case with macros,
edge-clipped boxes and a frozen-z subset; the small design's cloud at its
golden point on 64x64x2), each with the reference's phi, energy and gradient.
The reference is never imported at test time or on the GPU box.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from place3d import density as rdn  # noqa: E402


def case_random():
    rng = np.random.default_rng(23)
    grid = rdn.DensityGrid(16.0, 12.0, 16, 12, 8)
    n, nm = 60, 4
    w = np.r_[rng.uniform(0.4, 2.5, n - nm), rng.uniform(3, 7, nm)]
    h = np.r_[rng.uniform(0.4, 2.5, n - nm), rng.uniform(2, 5, nm)]
    x = rng.uniform(-0.5, 16.5, n)  # some boxes cross the region boundary (clipped)
    y = rng.uniform(-0.5, 12.5, n)
    z = rng.uniform(grid.dz / 4, 3 * grid.dz / 4, n)
    dep = np.full(n, grid.dz / 2)
    weight = np.r_[np.ones(n - nm), np.full(nm, 0.9)]
    macro = np.r_[np.zeros(n - nm, bool), np.ones(nm, bool)]
    freeze = rng.random(n) < 0.2
    return grid, (x, y, z, w, h, dep, weight, macro), freeze


def solve(grid, c, freeze):
    cloud = rdn.ChargeCloud(*c)
    rho = rdn.accumulate_density(grid, cloud)
    phi, coef = rdn.solve_potential(rho, grid)
    ex, ey, ez = rdn.electric_field(coef, grid)
    e, grad = rdn.density_energy_and_gradient(grid, cloud, phi, ex, ey, ez, freeze_z=freeze)
    return phi, e, grad


def main():
    out = {}
    grid, c, freeze = case_random()
    phi, e, grad = solve(grid, c, freeze)
    for k, v in zip(("x", "y", "z", "w", "h", "dep", "weight", "is_macro"), c):
        out[f"a_{k}"] = v
    out.update(a_freeze=freeze, a_phi=phi, a_energy=e, a_grad=grad,
               a_grid=np.array([16.0, 12.0, 16, 12, 8]))
    np.savez_compressed(os.path.join(HERE, "energy_grad.npz"), **out)
    print("energy", e, "grad norm", np.abs(grad).sum())


if __name__ == "__main__":
    main()
