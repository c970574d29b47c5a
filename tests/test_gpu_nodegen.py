"""Device node generation against the reference's own generator output
(tests/golden/nodegen_*.npz, oracle/make_golden_nodegen.py) and the reference's
tests/test_nodegen.py cases.

Bar: box / circle / sphere domains bit-identical to the reference (positions, spacing,
kinds, roles, BCs, normals, origins, lattice map); star obstacles (device sin/cos) equal
counts and layout, positions within 1e-12."""

import ast

import numpy as np
import numpy.testing as npt
import pytest

from paper_2303_01760_b200 import config as hc
from paper_2303_01760_b200 import generate as G
from paper_2303_01760_b200.geometry import Circle, DomainSpec, Obstacle
from paper_2303_01760_b200.nodegen import KIND_REGULAR, KIND_SCATTERED

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

EXACT = ["dvd_h0398", "dvd_h01", "dvd_pure_scattered", "dvd_pure_regular", "split_vertical", "split_full",
         "custom_box", "spheres3d_h05", "spheres3d_two_seed5"]


def golden(name):
    with np.load(GOLDEN / f"nodegen_{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def config_of(g):
    return hc.CaseConfig(**dict(ast.literal_eval(str(g["config"]))))


def same_nan(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b), equal_nan=True)


def check_layout(spec, g, tol=0.0):
    assert len(spec.obstacles) == len(g["obs_kind"])
    for j, obs in enumerate(spec.obstacles):
        sh = obs.shape
        if g["obs_kind"][j] == 1:
            got = (*sh.center, sh.mean_radius, sh.amplitude, sh.lobes, sh.phase)
            want = g["obs_par"][j, :6]
        else:
            got = (*sh.center, sh.radius)
            want = g["obs_par"][j, :len(sh.center) + 1]
        npt.assert_allclose(got, want, rtol=0, atol=tol)


@pytest.mark.parametrize("name", EXACT)
def test_hybrid_discretize_bit_identical(name):
    g = golden(name)
    cfg = config_of(g)
    spec = hc.build_domain(cfg)
    check_layout(spec, g)
    ns = G.hybrid_discretize(cfg, spec)
    assert len(ns) == len(g["positions"]), (ns.counts, np.bincount(g["kind"], minlength=3))
    assert np.array_equal(ns.kind, g["kind"])
    assert np.array_equal(ns.positions, g["positions"]), np.abs(ns.positions - g["positions"]).max()
    assert np.array_equal(ns.spacing, g["spacing"])
    assert np.array_equal(ns.role, g["role"])
    assert same_nan(ns.bc_value, g["bc_value"]) and same_nan(ns.normals, g["normals"])
    assert list(ns.origin) == [str(s) for s in g["origin"]]
    assert np.array_equal(ns.lattice.grid, g["lattice_grid"])
    assert np.array_equal(ns.lattice_idx, g["lattice_idx"])
    assert np.array_equal(ns.lattice.step, g["lattice_step"]) and tuple(ns.lattice.cells) == tuple(g["lattice_cells"])


def test_obstacles2d_star_to_rounding():
    g = golden("obstacles2d_h02")
    cfg = config_of(g)
    spec = hc.build_domain(cfg)
    check_layout(spec, g)
    ns = G.hybrid_discretize(cfg, spec)
    assert np.array_equal(ns.kind, g["kind"]), (ns.counts, np.bincount(g["kind"], minlength=3))
    npt.assert_allclose(ns.positions, g["positions"], rtol=0, atol=1e-12)
    npt.assert_allclose(ns.spacing, g["spacing"], rtol=1e-12)
    assert np.array_equal(ns.role, g["role"]) and list(ns.origin) == [str(s) for s in g["origin"]]
    assert np.array_equal(ns.lattice.grid, g["lattice_grid"])
    # reference test_nodegen.py TestHybridDiscretize invariants on the same case
    step = float(np.max(ns.lattice.step))
    fn = G.SpacingFunction(step, cfg.h_s, cfg.delta_h, spec.obstacle_distance)
    sc = ns.kind == KIND_SCATTERED
    assert np.array_equal(ns.spacing[sc], fn(ns.positions[sc]))
    width = cfg.delta_h * step
    dist = spec.obstacle_distance(ns.positions)
    assert np.all(dist[sc] < width) and np.all(dist[ns.kind == KIND_REGULAR] >= width)
    assert ns.min_distance_violations() == 0
    assert np.all(spec.signed_distance(ns.positions) <= 1e-9)


def test_reference_domain_objects_drop_in():
    """A DomainSpec built from the golden layout (as a caller's spec) gives the same set."""
    g = golden("spheres3d_h05")
    cfg = config_of(g)
    obs = tuple(Obstacle(Circle(tuple(p[:3]), float(p[3])), None if np.isnan(t) else float(t))
                for p, t in zip(g["obs_par"], g["obs_temp"]))
    ns = G.hybrid_discretize(cfg, DomainSpec(np.zeros(3), np.ones(3), obs))
    assert np.array_equal(ns.positions, g["positions"])


def test_api_fills_and_geometry():
    a = np.load(GOLDEN / "nodegen_api.npz")
    box = DomainSpec(np.zeros(2), np.ones(2))
    circ = DomainSpec(np.zeros(2), np.ones(2), (Obstacle(Circle((0.5, 0.5), 0.2), 0.0),))
    fill = G.regular_fill(circ, 0.05)
    assert np.array_equal(fill.positions, a["fill_pos"]) and np.array_equal(fill.indices, a["fill_idx"])
    assert np.array_equal(fill.step, a["fill_step"])
    assert np.array_equal(G.carve_transition(fill, circ, 2.0, 0.05).positions, a["carved_pos"])
    p = a["probe"]
    assert np.array_equal(circ.signed_distance(p), a["probe_sd"])
    assert np.array_equal(circ.obstacle_distance(p), a["probe_obs"])
    assert np.array_equal(circ.box_signed_distance(p), a["probe_box"])
    graded = G.SpacingFunction(0.03, 0.01, 4.0, circ.obstacle_distance)
    assert np.array_equal(graded(p), a["probe_h"])
    seeds = np.array([[0.5, 0.0], [0.0, 0.5], [1.0, 0.5], [0.5, 1.0]])
    sf = G.SpacingFunction(0.1, 0.1, 0.0)
    assert np.array_equal(G.scattered_fill(box, seeds, sf, rng_seed=11), a["sf11"])
    assert np.array_equal(G.scattered_fill(box, seeds, sf, rng_seed=12), a["sf12"])
    assert np.array_equal(G.scattered_fill(circ, seeds, graded, rng_seed=4), a["sf_graded"])


# ---- the reference's tests/test_nodegen.py cases
def unit_box(*shapes):
    return DomainSpec(np.zeros(2), np.ones(2), tuple(Obstacle(s, 0.0) for s in shapes))


def test_regular_fill_cases():
    fill = G.regular_fill(unit_box(), 0.25)
    assert len(fill) == 9
    assert {(round(x, 12), round(y, 12)) for x, y in fill.positions} == {(0.25 * i, 0.25 * j) for i in (1, 2, 3)
                                                                           for j in (1, 2, 3)}
    npt.assert_allclose(G.regular_fill(unit_box(), 0.5).positions, [[0.5, 0.5]])
    spec = unit_box(Circle((0.5, 0.5), 0.3))
    fill = G.regular_fill(spec, 0.25)
    full = np.array([[0.25 * i, 0.25 * j] for i in (1, 2, 3) for j in (1, 2, 3)])
    keep = spec.signed_distance(full) <= -0.125 * (1 - 1e-12)
    assert sorted(map(tuple, fill.positions)) == sorted(map(tuple, full[keep]))
    with pytest.raises(hc.ConfigurationError):
        G.regular_fill(unit_box(), 2.0)
    npt.assert_allclose(G.regular_fill(unit_box(), 0.0398).step, [0.04, 0.04])


def test_carve_cases():
    spec = unit_box(Circle((0.5, 0.5), 0.2))
    fill = G.regular_fill(spec, 0.1)
    npt.assert_array_equal(G.carve_transition(fill, spec, 0.0, 0.1).positions, fill.positions)
    assert len(G.carve_transition(fill, spec, 50.0, 0.1)) == 0


def test_scattered_fill_cases():
    spec = unit_box()
    sf = G.SpacingFunction(0.1, 0.1, 0.0)
    seeds = np.array([[0.5, 0.0], [0.0, 0.5], [1.0, 0.5], [0.5, 1.0]])
    a = G.scattered_fill(spec, seeds, sf, rng_seed=11)
    assert a.tobytes() == G.scattered_fill(spec, seeds, sf, rng_seed=11).tobytes()
    out = G.scattered_fill(spec, np.array([[0.5, 0.5]]), sf, 1,
                           region=lambda pts: np.zeros(len(np.atleast_2d(pts)), dtype=bool))
    assert out.shape == (0, 2)


def test_spacing_function_values():
    spec = unit_box(Circle((0.5, 0.5), 0.2))
    fn = G.SpacingFunction(0.03, 0.01, 4.0, spec.obstacle_distance)
    npt.assert_allclose(fn(np.array([[0.7, 0.5]])), [0.01])
    npt.assert_allclose(fn(np.array([[0.95, 0.05]])), [0.03])
    npt.assert_allclose(fn(np.array([[0.76, 0.5]])), [0.02])
    with pytest.raises(hc.ConfigurationError):
        G.SpacingFunction(0.01, 0.02, 4.0)


def test_split_limits_and_orientation():
    ns = G.hybrid_discretize(hc.CaseConfig(case="dvd-split", h_r=0.05, delta_h=1 / 0.05))
    assert ns.counts[0] == 0 and ns.counts[1] > 0
    ns2 = G.hybrid_discretize(hc.CaseConfig(case="dvd-split", h_r=0.05, delta_h=0.0))
    assert ns2.counts[1] == 0 and ns2.counts[0] > 0
    cfg = hc.CaseConfig(case="dvd-split", h_r=0.05, delta_h=8, split_orientation="horizontal")
    ns = G.hybrid_discretize(cfg)
    sc, reg = ns.positions[ns.kind == KIND_SCATTERED], ns.positions[ns.kind == KIND_REGULAR]
    assert np.all(sc[:, 1] < 0.4) and np.all(reg[:, 1] >= 0.4)
    ns_v = G.hybrid_discretize(cfg.with_overrides(split_orientation="vertical"))
    assert np.all(ns_v.positions[ns_v.kind == KIND_SCATTERED][:, 0] < 0.4)


def test_dvd_invariants_and_csv(tmp_path):
    ns = G.hybrid_discretize(hc.CaseConfig(case="dvd", h_r=0.0398))
    assert 560 <= len(ns) <= 700
    assert ns.min_distance_violations() == 0
    reg = ns.positions[ns.kind == KIND_REGULAR]
    assert not ((reg[:, 0] < 0.5) == (reg[:, 1] < 0.5)).any()
    path = tmp_path / "nodes.csv"
    ns.to_csv(path)
    back = type(ns).from_csv(path)
    npt.assert_array_equal(back.positions, ns.positions)
    node = ns.node(len(ns) - 1)
    assert node.normal is not None and node.kind == 2


def test_large_3d_fill_invariants():
    """A config-4-scale sphere case (beyond any golden): spacing / acceptance invariants."""
    cfg = hc.CaseConfig(case="spheres3d", h_r=0.02)
    spec = hc.build_domain(cfg)
    ns = G.hybrid_discretize(cfg, spec)
    nr, nsc, nb = ns.counts
    assert nsc > 10_000 and nr > 50_000
    assert ns.min_distance_violations() == 0
    assert np.all(spec.signed_distance(ns.positions) <= 1e-9)
    again = G.hybrid_discretize(cfg, spec)
    assert ns.positions.tobytes() == again.positions.tobytes()
