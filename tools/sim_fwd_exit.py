"""K6 lockstep steps with and without a warp-level early exit inside a batch (CPU cost model;
needs the oracle build).  A warp walks, per 128-record batch, the longest list of its alive
sub-quarters; with the exit it stops once all 128 of its pixels have terminated (checked every
`chk` steps).  Usage: PYTHONPATH=. python tools/sim_fwd_exit.py [n] [view] [n_views] [t_min]"""
import sys

import numpy as np

import oracle as O
from paper_2403_14244_b200 import isg

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
view = int(sys.argv[2]) if len(sys.argv) > 2 else 0
nv = int(sys.argv[3]) if len(sys.argv) > 3 else 1
t_min = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-5
W, H, B = 1920, 1080, 128
ms, co = isg.synth_scene(n, W, H, seed=2403)
cam = isg.Camera.synthetic(W, H, view, nv)
keys, vals, ranges, nvis = O.bin32(ms, co, cam)
img, tl, npr, cnt = O.render32(ms, co, cam, t_min=t_min, want_state=True)
R = np.asarray(cam.rotation, np.float64).reshape(3, 3)
t = np.asarray(cam.translation, np.float64)
pc = ms[:, :3].astype(np.float64) @ R.T + t
f = cam.focal
cx, cy = cam.principal_point
u = f * pc[:, 0] / pc[:, 2] + cx
v = f * pc[:, 1] / pc[:, 2] + cy
s = ms[:, 3] * f / pc[:, 2]
r2m = 9 * s * s
tx_n, ty_n = (W + 15) // 16, (H + 15) // 16
tile = (keys >> 32).astype(np.int64)
pos = np.arange(len(keys)) - ranges[tile, 0]
g = vals.astype(np.int64)
tx, ty = tile % tx_n, tile // tx_n
# per pixel: entry index after which it is terminated (inf if it never terminates).  The
# oracle's `tl` is the transmittance before the last contributor: one more factor gives the
# final transmittance.
INF = 1 << 40
yy, xx = np.mgrid[0:H, 0:W]
ptile = (yy // 16) * tx_n + xx // 16
has = npr > 0
gl = vals[np.minimum(ranges[ptile, 0].astype(np.int64) + npr.astype(np.int64) - 1,
                     len(vals) - 1)].astype(np.int64)
d2 = (xx + 0.5 - u[gl]) ** 2 + (yy + 0.5 - v[gl]) ** 2
alpha = co[gl, 3] * np.exp(-d2 / (2 * s[gl] ** 2))
t_fin = np.where(has, tl * (1 - alpha), 1.0)
print(f"terminated pixels {(t_fin <= t_min).mean():.3f}")
endp = np.where(t_fin <= t_min, npr.astype(np.int64), INF)
E = np.full((ty_n * 16, tx_n * 16), -1, np.int64)  # padding pixels: terminated from the start
E[:H, :W] = endp
# per (tile, warp): warp w = rows 8w..8w+7 of the tile
Ew = E.reshape(ty_n, 2, 8, tx_n, 16).max(axis=(2, 4))  # [ty, w, tx]
# per sub-quarter (for alive-at-batch-start)
Esq = E.reshape(ty_n, 4, 4, tx_n, 4, 4).max(axis=(2, 5))  # [ty, r4, tx, c4]
rel = np.zeros((len(g), 16), bool)
for r4 in range(4):
    y0 = ty * 16 + 4 * r4 + 0.5
    y1 = np.minimum(ty * 16 + 4 * r4 + 4, H) - 1 + 0.5
    dy = np.clip(v[g], y0, y1) - v[g]
    for c4 in range(4):
        x0 = tx * 16 + 4 * c4 + 0.5
        x1 = np.minimum(tx * 16 + 4 * c4 + 4, W) - 1 + 0.5
        dx = np.clip(u[g], x0, x1) - u[g]
        rel[:, 4 * r4 + c4] = ((dx * dx + dy * dy <= r2m[g]) & (ty * 16 + 4 * r4 < H) &
                               (tx * 16 + 4 * c4 < W))
batch = pos // B
bstart = batch * B
# group alive at batch start: some pixel not terminated before bstart
alive = np.zeros((len(g), 16), bool)
for r4 in range(4):
    for c4 in range(4):
        alive[:, 4 * r4 + c4] = Esq[ty, r4, tx, c4] > bstart
rel_a = rel & alive
key = tile * 100000 + batch
uk, inv = np.unique(key, return_inverse=True)
tb, bb = uk // 100000, uk % 100000
for chk in (1, 4, 8):
    tot0 = tot1 = 0
    for w in range(2):
        cols = [4 * r4 + c4 for r4 in (2 * w, 2 * w + 1) for c4 in range(4)]
        Ewe = Ew[ty, w, tx]  # per entry: the warp's exit entry
        C0 = np.zeros((len(uk), 8), np.int64)
        C1 = np.zeros((len(uk), 8), np.int64)
        for k, col in enumerate(cols):
            C0[:, k] = np.bincount(inv, weights=rel_a[:, col], minlength=len(uk))
            C1[:, k] = np.bincount(inv, weights=rel_a[:, col] & (pos < Ewe), minlength=len(uk))
        s0 = C0.max(1)
        s1 = np.minimum(s0, ((C1.max(1) + chk - 1) // chk) * chk)
        # the CTA-level stop: batches at or past both warps' exits are skipped entirely
        tot0 += s0.sum()
        tot1 += s1.sum()
    if chk == 1:
        print(f"n {n} view {view}/{nv}: warp steps {tot0:,}")
    print(f"  with a warp exit checked every {chk} steps: {tot1:,} ({tot1 / tot0:.3f})")
