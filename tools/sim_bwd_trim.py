"""Where K7's walk slots go (CPU cost model; needs the oracle build).

Bins a scene with the FP32 oracle and, for every tile, takes the entries K7 walks in batches of
128 (reverse depth order), the 4x4 sub-quarter relevance masks the forward writes and each
sub-quarter's own last processed entry (lists trimmed there, as K7 does).  Reports, in pixel
slots (one warp step = 8 groups x 16 pixels = 128 slots):
  lockstep  : sum over (tile, batch, warp) of the longest of the warp's 8 lists
  per group : sum of the lists themselves (no lockstep padding)
  active    : pixel-entry pairs that are in the circle and before the pixel's last entry
Usage: PYTHONPATH=. python tools/sim_bwd_trim.py [n] [view] [n_views] [t_min]"""
import sys

import numpy as np

import oracle as O
from paper_2403_14244_b200 import isg

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
view = int(sys.argv[2]) if len(sys.argv) > 2 else 0
nv = int(sys.argv[3]) if len(sys.argv) > 3 else 1
t_min = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-5
W, H = 1920, 1080
B = int(__import__("os").environ.get("SIM_BATCH", 128))
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
npr_p = np.zeros((ty_n * 16, tx_n * 16), np.int64)
npr_p[:H, :W] = npr
m = npr_p.reshape(ty_n, 16, tx_n, 16).max(axis=(1, 3)).reshape(-1)
pos = np.arange(len(keys)) - ranges[tile, 0]
keep = pos < m[tile]
tile, pos, g = tile[keep], pos[keep], vals[keep].astype(np.int64)
tx, ty = tile % tx_n, tile // tx_n
print(f"n {n} view {view}/{nv} t_min {t_min}: keys {len(keys)}, walked entries {len(g)}")
# sub-quarter max processed count (trim) and the relevance mask
sqmax = npr_p.reshape(ty_n, 4, 4, tx_n, 4, 4).max(axis=(2, 5))  # [ty, r4, tx, c4]
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
                               (tx * 16 + 4 * c4 < W) & (pos < sqmax[ty, r4, tx, c4]))
# K7's sub index: sub = 8 w + gq, q = sub >> 2 (quarter: 8x8), sq = sub & 3 -> (r4, c4)
order = []
for sub in range(16):
    q, sq = sub >> 2, sub & 3
    r4 = (q >> 1) * 2 + (sq >> 1)
    c4 = (q & 1) * 2 + (sq & 1)
    order.append(4 * r4 + c4)
rel = rel[:, order]
batch = (m[tile] - 1 - pos) // B
key = tile * 100000 + batch
uk, inv = np.unique(key, return_inverse=True)
C = np.zeros((len(uk), 16), np.int64)
for k in range(16):
    C[:, k] = np.bincount(inv, weights=rel[:, k], minlength=len(uk))
lock = C[:, :8].max(1).sum() + C[:, 8:].max(1).sum()
per = C.sum() / 8
# active pixel pairs: in circle and before the pixel's own last entry (per-pixel check)
act = 0
for r in range(16):
    for c in range(16):
        y = ty * 16 + r
        x = tx * 16 + c
        ok = (y < H) & (x < W)
        yy, xx = np.minimum(y, H - 1), np.minimum(x, W - 1)
        dx = xx + 0.5 - u[g]
        dy = yy + 0.5 - v[g]
        act += int((ok & (dx * dx + dy * dy <= r2m[g]) & (pos < npr[yy, xx])).sum())
print(f"warp steps lockstep {lock:,} ({lock * 128:,} slots); no padding {per:,.0f}; "
      f"active pairs {act:,} ({act / (lock * 128):.2f} of the slots, "
      f"{act / (per * 128):.2f} without padding)")

# warp assignment by the sub-quarters' last entries: the 8 deepest-terminating sub-quarters of
# a tile share warp 0, so a long list pads the lockstep of fewer short ones
sq16 = sqmax.transpose(0, 2, 1, 3).reshape(ty_n * tx_n, 16)[:, order]  # per tile, K7 sub order
rank_perm = np.argsort(-sq16, axis=1, kind="stable")  # [tile, slot] -> sub
tb = uk // 100000
Cs = np.take_along_axis(C, rank_perm[tb], axis=1)
lock_s = Cs[:, :8].max(1).sum() + Cs[:, 8:].max(1).sum()
print(f"sorted by sub-quarter depth: lockstep {lock_s:,} warp steps ({lock_s / lock:.3f} of K7's)")
# and by the tile's total relevant entries per sub-quarter (an oracle bound for any static map)
G = np.zeros((ty_n * tx_n, 16), np.int64)
np.add.at(G, tb, C)
Cg = np.take_along_axis(C, np.argsort(-G, axis=1, kind="stable")[tb], axis=1)
lock_g = Cg[:, :8].max(1).sum() + Cg[:, 8:].max(1).sum()
print(f"sorted by relevant entries: lockstep {lock_g:,} warp steps ({lock_g / lock:.3f})")

# one batch of lookahead: a group whose list of the current batch is done walks on into its
# list of the next staged batch while the warp's longest list finishes
nb = np.zeros(len(uk), np.int64)
tile_of = uk // 100000
b_of = uk % 100000
tot_la = 0
tot_lock = 0
order_rows = np.lexsort((b_of, tile_of))
rows_t = tile_of[order_rows]
bounds = np.flatnonzero(np.diff(rows_t)) + 1
for seg in np.split(order_rows, bounds):
    Cseg = C[seg]  # batches of one tile, in walk order (batch 0 = the top of the list)
    for w in range(2):
        L = Cseg[:, 8 * w:8 * w + 8].astype(np.int64)
        rem = L[0].copy()
        for b in range(len(L)):
            steps = rem.max()
            tot_lock += L[b].max()
            tot_la += steps
            if b + 1 < len(L):
                adv = np.minimum(steps - rem, L[b + 1])
                rem = L[b + 1] - adv
print(f"one-batch lookahead: {tot_la:,} warp steps ({tot_la / tot_lock:.3f} of lockstep {tot_lock:,})")

# exact masks: a sub-quarter is listed for an entry only if one of its 16 pixel centres is
# inside the circle and the pixel has not finished before the entry (what K6 could record
# from its own walk instead of the closest-point box test)
ex = np.zeros((len(g), 16), bool)
for r4 in range(4):
    for c4 in range(4):
        hit = np.zeros(len(g), bool)
        for rr in range(4):
            for cc in range(4):
                y = ty * 16 + 4 * r4 + rr
                x = tx * 16 + 4 * c4 + cc
                ok = (y < H) & (x < W)
                yy, xx = np.minimum(y, H - 1), np.minimum(x, W - 1)
                d2 = (xx + 0.5 - u[g]) ** 2 + (yy + 0.5 - v[g]) ** 2
                hit |= ok & (d2 <= r2m[g]) & (pos < npr[yy, xx])
        ex[:, 4 * r4 + c4] = hit
ex = ex[:, order]
Ce = np.zeros((len(uk), 16), np.int64)
for k in range(16):
    Ce[:, k] = np.bincount(inv, weights=ex[:, k], minlength=len(uk))
lock_e = Ce[:, :8].max(1).sum() + Ce[:, 8:].max(1).sum()
print(f"exact per-sub-quarter masks: lockstep {lock_e:,} warp steps ({lock_e / lock:.3f} of the box masks'); "
      f"listed group-entries {ex.sum():,} vs {rel.sum():,}")
