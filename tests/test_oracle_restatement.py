"""Pin the plain-C restatement (oracle/lfd_oracle.c) against the reference (oracle/_ref) and
the frozen golden vectors: SLIC labels/records/CSR, sweep winners, rasterize and three refine
iterations with the accepted counts, bit for bit, on C1 and on a grid-rig / staircase scene."""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run_port(sc, S, L, iters):
    from oracle.port import Port

    P = Port(sc["lab"], sc["cams"], sc["range"])
    V = P.V
    for v in range(V):
        P.slic(v, S, 0.1, 10)
    planes = np.stack([P.sweep(v, L, 0.05, 0, 0) for v in range(V)])
    depth = np.stack([P.rasterize(v, planes[v]) for v in range(V)])
    step = (1.0 / sc["range"][0] - 1.0 / sc["range"][1]) / (L - 1)
    sigma, size_init = 1.5 * step, min(P.W, P.H)
    hist = [(planes.copy(), depth.copy(), 0)]
    for l in range(1, iters + 1):
        planes, acc = P.refine_iteration(l, planes, depth, sigma, size_init)
        depth = np.stack([P.rasterize(v, planes[v]) for v in range(V)])
        hist.append((planes.copy(), depth.copy(), acc))
    return P, hist


def test_port_matches_c1_golden():
    from oracle.port import Port  # noqa: F401
    from paper_1812_06856_b200 import scenes

    g = np.load(os.path.join(ROOT, "tests", "golden", "c1_golden.npz"))
    sc = scenes.render_scene("cluttered", 3, 320, 240, 320.0, 0.1)
    P, hist = _run_port(sc, 12, 32, 3)
    for v in range(3):
        assert np.array_equal(P.grids[v].labels, g[f"labels{v}"])
        assert np.array_equal(hist[0][0][v], g[f"sweep{v}"])
    for l in range(1, 4):
        assert hist[l][2] == g["accepted"][l - 1], f"accepted differs at l={l}"
        for v in range(3):
            assert np.array_equal(hist[l][0][v], g[f"refine{l}_{v}"]), f"planes differ l={l} v={v}"
    for v in range(3):
        assert np.array_equal(hist[3][1][v], g[f"depth{v}"])


@pytest.mark.parametrize("kind,n,w,h,f,b,grid,S,L", [
    ("cluttered", 4, 128, 96, 128.0, 0.05, (2, 2), 8, 12),
    ("staircase", 3, 96, 72, 80.0, 0.4, (0, 0), 10, 16),
])
def test_port_matches_reference(ref, kind, n, w, h, f, b, grid, S, L):
    sc = ref.render_scene(kind, n, w, h, f, b, 0.0, grid)
    P, hist = _run_port(sc, S, L, 2)
    rs = ref.Session(sc["lab"], sc["cams"], sc["range"])
    V = sc["lab"].shape[0]
    for v in range(V):
        rs.slic(v, S, 0.1, 10)
        want = rs.grid(v)
        assert np.array_equal(P.grids[v].labels, want["labels"])
        assert np.array_equal(P.grids[v].off, want["offsets"]) and np.array_equal(P.grids[v].mem, want["members"])
        assert np.array_equal(P.grids[v].rec["cx"], want["records"]["cx"])
        assert np.array_equal(P.grids[v].rec["color"], want["records"]["color"])
        assert np.array_equal(hist[0][0][v], rs.sweep(v, L, 0.05, 0, 0))
    rs.rasterize()
    rs.refine_context(L, iterations=2)
    for l in (1, 2):
        acc, _ = rs.refine_iteration(l, with_stats=True)
        rs.rasterize()
        assert acc == hist[l][2]
        for v in range(V):
            assert np.array_equal(hist[l][0][v], rs.planes(v))
            assert np.array_equal(hist[l][1][v], rs.depth(v))
