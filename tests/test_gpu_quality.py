"""the paper's reconstruction-quality experiments
(§5.1) as regression tests, end to end on the GPU: density measures
(rbf_density) choose sigma by Eq. 9 / Eq. 10-11, the system is solved, the
interpolant is evaluated on a grid and its eps-masked zero set extracted.

Stand-in data: the paper's "widely scattered" 382-point cloud of
the unit sphere is not available; a seeded i.i.d. uniform sample of 382 points
plays its role.  Quality of a reconstruction = the largest holes (99th percentile
distance from the true surface to the zero set) and the median radial error of
the zero-set points.  What the paper shows and these
tests pin:
  * sigma = 2 q_X (Eq. 9) "interpolates the cloud but the quality is totally
    unsatisfactory"; sigma = sqrt(2) h_{X,M} (Eq. 10-11) reconstructs the sphere;
  * 50% of the points: sqrt(2) h of the reduced cloud (recomputed fill distance)
    reconstructs the sphere and beats sqrt(2) h of the full cloud (with this
    stand-in the full-cloud sigma degrades the surface instead of breaking it);
  * the upper semi-sphere with sigma = sqrt(2) h_{X,M+} reconstructs M+ only.
"""
import numpy as np
import pytest
import torch

from synth.surfaces import fibonacci_sphere

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no CPU fallback)"
    import paper_1305_5179_b200 as R
    R.load_library()
    return R


@pytest.fixture(scope="module")
def ctx(R):
    return R.Context(0)


def _cloud(n=382, seed=11, jitter=0.03):
    """Fibonacci lattice with seeded Gaussian jitter, projected back on the sphere:
    scattered (close pairs: small q_X) but covering (fill distance near the
    lattice's) -- the regime of the paper's 382-point cloud (q ~ 0.024, h ~ 0.11)."""
    f, _ = fibonacci_sphere(n)
    v = f + jitter * np.random.default_rng(seed).normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def _dev(a, dt=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")


def reconstruct(R, ctx, x, sigma, grid_n=72, box=1.6):
    """Alg. 1 with the library: extend (delta = 0.1 sigma, reading R4), solve, grid, zero set."""
    delta = 0.1 * sigma
    centres, b = R.extend_points(ctx, _dev(x), _dev(x), delta)     # unit sphere: normal = x
    kern = R.Kernel(sigma)
    cells = R.Cells(ctx, centres, kern)
    # shifted block-Jacobi (finding F4: robust for any sigma/spacing), fixed budget
    w, rep = R.gmres_solve(ctx, cells, kern, b, restart=50, rtol=1e-6, kind=1, core_target=64, shift=0.003,
                           local_fp32=1, max_iters=150)
    lo, hi, gn = (-box,) * 3, (box,) * 3, (grid_n,) * 3
    F = R.eval_grid(ctx, cells, kern, w, lo, hi, gn)
    pts = R.zero_set(ctx, F.reshape(-1), lo, hi, gn, _dev(x), 2 * sigma).cpu().numpy()
    return pts, rep


def quality(pts, upper_only=False):
    """(hole, err): hole = 99th percentile over 20000 points of the true surface of
    the distance to the nearest zero-set point (a gap in the reconstruction shows
    up as a large hole); err = median | |p| - 1 | of the zero-set points."""
    from scipy.spatial import cKDTree
    truth, _ = fibonacci_sphere(20000)
    if upper_only:
        truth = truth[truth[:, 2] > 0.1]
        pts = pts[pts[:, 2] > 0.1]
    if len(pts) == 0:
        return np.inf, np.inf
    hole = float(np.quantile(cKDTree(pts).query(truth)[0], 0.99))
    return hole, float(np.median(np.abs(np.linalg.norm(pts, axis=1) - 1.0)))


def fill_on_sphere(R, ctx, x, upper_only=False):
    om, _ = fibonacci_sphere(20000)
    if upper_only:
        om = om[om[:, 2] >= 0]
    return R.density(ctx, _dev(x), _dev(om))


STEP = 3.2 / 71   # grid spacing of reconstruct(): a closed surface leaves holes < ~1 step


def test_sigma_choice_on_scattered_sphere(R, ctx):
    x = _cloud()
    dens = fill_on_sphere(R, ctx, x)
    hole_s, err_s = quality(reconstruct(R, ctx, x, dens["sigma_q"])[0])   # Eq. 9: sigma = 2 q_X
    hole_g, err_g = quality(reconstruct(R, ctx, x, dens["sigma_h"])[0])   # Eq. 10: sigma = sqrt(2) h_{X,M}
    print(f"sigma_q={dens['sigma_q']:.4f} hole={hole_s:.3f} err={err_s:.2e} | "
          f"sigma_h={dens['sigma_h']:.4f} hole={hole_g:.3f} err={err_g:.2e}")
    assert dens["sigma_q"] < dens["sigma_h"]
    assert hole_g <= STEP and err_g <= 1e-3                       # the sphere, closed
    assert hole_s >= 1.5 * hole_g and err_s >= 10 * err_g         # "totally unsatisfactory": gaps, bumps


def test_incomplete_data_needs_recomputed_fill_distance(R, ctx):
    x = _cloud()
    half = x[np.random.default_rng(5).permutation(len(x))[: len(x) // 2]]
    s_full = fill_on_sphere(R, ctx, x)["sigma_h"]
    s_half = fill_on_sphere(R, ctx, half)["sigma_h"]
    old = quality(reconstruct(R, ctx, half, s_full)[0])
    new = quality(reconstruct(R, ctx, half, s_half)[0])
    print(f"half cloud: sigma_full={s_full:.4f} hole={old[0]:.3f} err={old[1]:.2e} | "
          f"sigma_half={s_half:.4f} hole={new[0]:.3f} err={new[1]:.2e}")
    assert s_half > s_full
    assert new[0] <= STEP and new[1] <= 1e-3
    assert new[1] <= 0.5 * old[1]                                 # the recomputed fill distance is better


def test_semi_sphere(R, ctx):
    x = _cloud(764, seed=3)
    x = x[x[:, 2] >= 0]
    s_plus = fill_on_sphere(R, ctx, x, upper_only=True)["sigma_h"]
    pts = reconstruct(R, ctx, x, s_plus)[0]
    hole, err = quality(pts, upper_only=True)
    print(f"semi-sphere: sigma={s_plus:.4f} hole={hole:.3f} err={err:.2e}, lowest z={pts[:, 2].min():.3f}")
    assert hole <= STEP and err <= 1e-3
    assert pts[:, 2].min() >= -2.0 * s_plus * 1.05                # M+ only (within the eps mask of the rim)
