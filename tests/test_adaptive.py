"""Adaptive control: prune / merge / split of the splat set,
/root/reference/proj/src/optimize.cpp:150-284.

CPU: the oracle's control flow (oracle/isg_oracle.c or_adaptive_control) run with the
reference's own 2D rules is compared with the reference's compiled adaptive_control
(oracle/_ref) — bit-exact for prune and merge; split structure (the reference draws its split
directions from std::mt19937_64); 3D-rule properties (identity, cap, mass conservation).
GPU: k_adapt.cu through the C-ABI against the 3D oracle, bit-exact (FP64 rules rounded once).
"""
import numpy as np
import pytest

import oracle as O
from paper_2403_14244_b200 import isg


def have_ref():
    try:
        O.ref_lib()
        return True
    except RuntimeError:
        return False


def scene2d(rng, n, clusters=True):
    rec = np.zeros((n, 6))
    rec[:, 0:2] = rng.uniform(0, 40, (n, 2))
    rec[:, 2] = np.exp(rng.uniform(np.log(0.3), np.log(6.0), n))
    rec[:, 3:6] = rng.uniform(-0.05, 0.4, (n, 3))
    if clusters:  # near-duplicates that qualify for merging
        k = n // 3
        src = rng.integers(0, n, k)
        rec[:k] = rec[src] + np.concatenate([rng.normal(0, 0.05, (k, 2)), np.zeros((k, 1)),
                                             rng.normal(0, 0.01, (k, 3))], 1)
    return rec


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_2d_control_flow_matches_reference_prune_merge(seed):
    rng = np.random.default_rng(seed)
    n = 300
    rec = scene2d(rng, n)
    rec[rng.random(n) < 0.1, 3:6] *= 1e-3  # prunable
    args = (1e-2, 0.8, 0.1)
    ref = O.ref_adaptive_control_2d(rec, *args, split_sigma_max=1e9, max_particles=2 * n)
    out, (pruned, merged, split) = O.adaptive_control(
        rec, O.AdaptParams(*args, 1e9, 2 * n), dims=2)
    assert merged > 0 and pruned > 0 and split == 0
    np.testing.assert_array_equal(out, ref)


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_2d_prune_keeps_best_and_refused_merge_matches_reference():
    rng = np.random.default_rng(5)
    rec = scene2d(rng, 50, clusters=False)
    rec[:, 3:6] = rng.uniform(0, 1e-4, (50, 3))  # everything below the threshold
    ref = O.ref_adaptive_control_2d(rec, 1e-2, 0.5, 0.05, 1e9, 100)
    out, _ = O.adaptive_control(rec, O.AdaptParams(1e-2, 0.5, 0.05, 1e9, 100), dims=2)
    np.testing.assert_array_equal(out, ref)
    assert out.shape[0] == 1
    # zero-luminance pair: merge refused (optimize.cpp:205), both consumed, both kept
    a = np.array([[5.0, 5.0, 2.0, 0.5, -0.5 * 0.2126 / 0.7152, 0.0],
                  [5.1, 5.0, 2.0, 0.5, -0.5 * 0.2126 / 0.7152, 0.0]])
    ref = O.ref_adaptive_control_2d(a, 1e-3, 0.5, 0.05, 1e9, 4)
    out, (_, merged, _) = O.adaptive_control(a, O.AdaptParams(1e-3, 0.5, 0.05, 1e9, 4), dims=2)
    np.testing.assert_array_equal(out, ref)
    assert merged == 0 and out.shape[0] == 2


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_2d_split_structure_matches_reference():
    rng = np.random.default_rng(9)
    n = 120
    rec = scene2d(rng, n, clusters=False)
    cap = n + 17  # budget binds: widest first, ties by higher index
    ref = O.ref_adaptive_control_2d(rec, 0.0, 1e-9, 0.0, 2.0, cap)
    out, (_, _, split) = O.adaptive_control(rec, O.AdaptParams(0.0, 1e-9, 0.0, 2.0, cap), dims=2)
    assert out.shape == ref.shape and split == 17
    np.testing.assert_array_equal(out[:, 2:], ref[:, 2:])  # sigma, amplitudes, order
    moved = np.flatnonzero(np.any(out[:n, :2] != rec[:, :2], axis=1))
    assert len(moved) == 17
    for res in (out, ref):  # twins: child k pairs with the k-th widest parent, |a - b| = sigma
        for k, i in enumerate(moved[np.argsort(-rec[moved, 2] - 1e-12 * moved)]):
            d = np.linalg.norm(res[i, :2] - res[n + k, :2])
            assert d == pytest.approx(rec[i, 2], rel=1e-12)


def scene3d(rng, n, W=160, H=120, clusters=True):
    ms, co, cam = None, None, None
    f = 1000.0 * W / 1920.0
    z = rng.uniform(2, 10, n)
    u, v = rng.uniform(0, W, n), rng.uniform(0, H, n)
    s2d = np.exp(rng.uniform(np.log(0.5), np.log(16.0), n))  # several octaves -> grid levels
    ms = np.stack([(u - W / 2) * z / f, (v - H / 2) * z / f, z, s2d * z / f], 1)
    co = np.concatenate([rng.uniform(0, 1, (n, 3)), rng.uniform(0.0, 1.0, (n, 1))], 1)
    if clusters:
        k = n // 3
        src = rng.integers(0, n, k)
        ms[:k] = ms[src] + np.concatenate([rng.normal(0, 1, (k, 3)) * 0.05 * ms[src, 3:4],
                                           rng.uniform(-0.1, 0.1, (k, 1)) * ms[src, 3:4]], 1)
        co[:k, :3] = np.clip(co[src, :3] + rng.normal(0, 0.01, (k, 3)), 0, 1)
    co[rng.random(n) < 0.05, 3] = rng.uniform(0, 1e-3, 1)[0]  # prunable
    return ms.astype(np.float32), co.astype(np.float32)


def oracle3d(ms, co, prm, seed=0, round_=0):
    rec = np.concatenate([ms, co], 1).astype(np.float64)
    out, counts = O.adaptive_control(rec, O.AdaptParams(prm.prune_threshold,
                                                        prm.merge_distance_factor,
                                                        prm.merge_color_tol, prm.split_sigma_max,
                                                        prm.max_particles),
                                     dims=3, seed=seed, round_=round_)
    return out[:, :4].astype(np.float32), out[:, 4:].astype(np.float32), counts


def test_3d_oracle_properties():
    rng = np.random.default_rng(1)
    ms, co = scene3d(rng, 400)
    # nothing qualifies -> identity
    prm = isg.AdaptParams(0.0, 1e-12, 0.0, 1e9, 800)
    m2, c2, counts = oracle3d(ms, co, prm)
    assert counts == (0, 0, 0)
    np.testing.assert_array_equal(m2, ms)
    np.testing.assert_array_equal(c2, co)
    # cap respected, splits widest first, twins sigma/2 either side
    prm = isg.AdaptParams(0.0, 1e-12, 0.0, 0.02, 450)
    m2, c2, counts = oracle3d(ms, co, prm)
    assert m2.shape[0] == 450 and counts[2] == 50
    parents = np.argsort(-ms[:, 3].astype(np.float64) - 1e-9 * np.arange(400))[:50]
    for k, i in enumerate(sorted(parents, key=lambda i: (-ms[i, 3], -i))):
        d = np.linalg.norm(m2[i, :3].astype(np.float64) - m2[400 + k, :3])
        assert d == pytest.approx(ms[i, 3], rel=1e-5)
        assert m2[i, 3] == np.float32(np.float64(ms[i, 3]) * np.sqrt(0.5))
    # merge conserves footprint mass o sigma^2 (when the merged opacity stays < 1)
    a = np.array([[0, 0, 5, 0.1], [0.001, 0, 5, 0.12]], np.float32)
    c = np.array([[0.5, 0.5, 0.5, 0.2], [0.51, 0.5, 0.5, 0.3]], np.float32)
    m2, c2, counts = oracle3d(a, c, isg.AdaptParams(0.0, 0.5, 0.05, 1e9, 4))
    assert counts[1] == 1 and m2.shape[0] == 1
    mass = lambda m, c: float(c[:, 3].astype(np.float64) @ m[:, 3].astype(np.float64) ** 2)
    assert mass(m2, c2) == pytest.approx(mass(a, c), rel=1e-6)


# ---- GPU ------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def rend():
    r = isg.Renderer(0)
    yield r
    r.close()


CASES = [
    ("merge", 3000, isg.AdaptParams(1e-3, 0.5, 0.05, 1e9, 0)),
    ("merge_wide", 3000, isg.AdaptParams(1e-3, 2.0, 0.2, 1e9, 0)),
    ("split_cap", 2000, isg.AdaptParams(1e-3, 0.5, 0.05, 0.05, 2300)),
    ("all", 20000, isg.AdaptParams(1e-2, 1.0, 0.1, 0.08, 0)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("name,n,prm", CASES, ids=[c[0] for c in CASES])
def test_gpu_adaptive_control_matches_oracle(rend, name, n, prm):
    rng = np.random.default_rng(sum(name.encode()))
    ms, co = scene3d(rng, n)
    rend.set_scene(ms, co)
    res = rend.adaptive_control(prm, seed=77, round_=3)
    cap = prm.max_particles if prm.max_particles > 0 else 2 * n
    om, oc, counts = oracle3d(ms, co, isg.AdaptParams(prm.prune_threshold,
                                                      prm.merge_distance_factor,
                                                      prm.merge_color_tol, prm.split_sigma_max,
                                                      cap), seed=77, round_=3)
    gm, gc = rend.get_scene()
    assert (res["n_pruned"], res["n_merged"], res["n_split"]) == counts
    assert res["n_after"] == om.shape[0] == gm.shape[0]
    np.testing.assert_array_equal(gm, om)
    np.testing.assert_array_equal(gc, oc)
    if name != "split_cap":
        assert counts[1] > 0


@pytest.mark.gpu
def test_gpu_prune_all_keeps_best_and_training_continues(rend):
    rng = np.random.default_rng(3)
    W, H = 96, 72
    ms, co = scene3d(rng, 500, W, H, clusters=False)
    co[:, 3] = rng.uniform(0, 1e-4, 500).astype(np.float32)
    co[123, 3] = np.float32(2e-4)
    rend.set_scene(ms, co)
    res = rend.adaptive_control(isg.AdaptParams(1e-2, 0.5, 0.05, 1e9, 0))
    assert res["n_after"] == 1
    gm, gc = rend.get_scene()
    np.testing.assert_array_equal(gm[0], ms[123])
    # a full step still works on the new set, with more splats after a split round
    ms, co = scene3d(rng, 800, W, H)
    rend.set_scene(ms, co)
    res = rend.adaptive_control(isg.AdaptParams(1e-3, 0.5, 0.05, 0.05, 1200), seed=1)
    assert res["n_split"] > 0 and rend.n == res["n_after"] <= 1200
    cam = isg.Camera.synthetic(W, H)
    tms, tco = isg.synth_scene(800, W, H, seed=9)
    target = O.render32(tms, tco, cam)
    gm, gc = rend.get_scene()
    loss = rend.loss_backward(cam, target)
    loss_ref, g_ref = O.loss_backward32(gm, gc, cam, target)
    assert loss == pytest.approx(loss_ref, rel=1e-5)
    rend.adam_step(isg.AdamConfig())
    assert rend.stats()["adam_steps"] == 1


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(8))
def test_gpu_adaptive_control_randomized(rend, seed):
    """Seeded random scenes and rule parameters: counts and the resulting splat set bit-exact
    against the 3D oracle."""
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(1, 6000))
    ms, co = scene3d(rng, n, clusters=bool(rng.integers(0, 2)))
    prm = isg.AdaptParams(prune_threshold=float(rng.choice([0.0, 1e-3, 0.05])),
                          merge_distance_factor=float(rng.uniform(0.05, 2.5)),
                          merge_color_tol=float(rng.uniform(0.0, 0.4)),
                          split_sigma_max=float(rng.choice([1e9, rng.uniform(0.02, 0.2)])),
                          max_particles=int(rng.choice([0, n + int(rng.integers(0, n + 1))])))
    rend.set_scene(ms, co)
    res = rend.adaptive_control(prm, seed=seed, round_=seed % 3)
    cap = prm.max_particles if prm.max_particles > 0 else 2 * n
    om, oc, counts = oracle3d(ms, co, isg.AdaptParams(prm.prune_threshold,
                                                      prm.merge_distance_factor,
                                                      prm.merge_color_tol, prm.split_sigma_max,
                                                      cap), seed=seed, round_=seed % 3)
    gm, gc = rend.get_scene()
    assert (res["n_pruned"], res["n_merged"], res["n_split"]) == counts
    np.testing.assert_array_equal(gm, om)
    np.testing.assert_array_equal(gc, oc)
