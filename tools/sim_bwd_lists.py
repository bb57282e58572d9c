"""Cost model for the blend backward's group layouts (run on CPU; needs the oracle build).

Bins the C3 scene with the FP32 oracle, takes every tile's walked entries in batches of 32
(the K7 staging), and counts per batch the entries relevant to each 4x4 sub-quarter.  The
lockstep cost of a layout is the per-batch maximum over the sub-quarters a warp owns, times an
estimated instruction count per warp step:
  v5 (2 warps x 8 four-lane groups, 4 px/lane) ~119 instr/step,
  v6 (1 warp x 16 two-lane groups, 8 px/lane)  ~174 instr/step,
  8x4 / 4x8 sub-blocks (1 warp x 8 four-lane groups, 8 px/lane) ~190 instr/step.
Measured: v6 has ~22% fewer instructions but 148 registers and twice the shared memory per
warp; it ran 2-4% slower than v5 on the B200, so K7 stays v5.
Usage: PYTHONPATH=. python tools/sim_bwd_lists.py"""
import numpy as np, oracle as O
from paper_2403_14244_b200 import isg
W,H,n=1920,1080,1_000_000
ms,co=isg.synth_scene(n,W,H,seed=2403)
cam=isg.Camera.synthetic(W,H)
keys,vals,ranges,nvis=O.bin32(ms,co,cam)
img,tl,npr,cnt=O.render32(ms,co,cam,want_state=True)
R=np.asarray(cam.rotation,np.float64).reshape(3,3); t=np.asarray(cam.translation,np.float64)
pc=ms[:,:3].astype(np.float64)@R.T+t
f=cam.focal; cx,cy=cam.principal_point if hasattr(cam,'principal_point') else (cam.cx,cam.cy)
u=f*pc[:,0]/pc[:,2]+cx; v=f*pc[:,1]/pc[:,2]+cy; s=ms[:,3]*f/pc[:,2]; r2m=9*s*s
tx_n=(W+15)//16; ty_n=(H+15)//16; T=tx_n*ty_n
tile=(keys>>32).astype(np.int64)
# m per tile = max npr over the tile's pixels
npr_p=np.zeros((ty_n*16,tx_n*16),np.int64); npr_p[:H,:W]=npr
m=npr_p.reshape(ty_n,16,tx_n,16).max(axis=(1,3)).reshape(-1)
pos=np.arange(len(keys))-ranges[tile,0]
keep=pos<m[tile]
tile=tile[keep]; pos=pos[keep]; g=vals[keep].astype(np.int64)
print('entries walked',len(g),'of',len(keys))
tx=tile%tx_n; ty=tile//tx_n
batch=(m[tile]-1-pos)//32
# 16 subs: sub index = 4*row4 + col4 (row4, col4 in 0..3)
cnts={}
rel=np.zeros((len(g),16),bool)
for r4 in range(4):
    y0=ty*16+4*r4+0.5; y1=np.minimum(ty*16+4*r4+4,H)-1+0.5
    dy=np.clip(v[g],y0,y1)-v[g]
    for c4 in range(4):
        x0=tx*16+4*c4+0.5; x1=np.minimum(tx*16+4*c4+4,W)-1+0.5
        dx=np.clip(u[g],x0,x1)-u[g]
        rel[:,4*r4+c4]=(dx*dx+dy*dy<=r2m[g])&(ty*16+4*r4<H)&(tx*16+4*c4<W)
# per (tile,batch) counts per sub
key=tile*100000+batch
uk,inv=np.unique(key,return_inverse=True)
C=np.zeros((len(uk),16),np.int64)
for s_ in range(16): C[:,s_]=np.bincount(inv,weights=rel[:,s_],minlength=len(uk))
top=C[:,:8].max(1); bot=C[:,8:].max(1); all16=C.max(1)
mean=C.mean(1)
print('sum top+bot',(top+bot).sum(),'sum max16',all16.sum(),'sum mean*2',(mean*2).sum(), 'total rel', C.sum())
print('v5 cost (119/step, 2 warps)', (top+bot).sum()*119/1e6, 'v6 cost (174/step)', all16.sum()*174/1e6)
# 2x2 px per lane / 4-lane groups but subs arranged by columns? alt: warp0 = left half
left=C[:,[0,1,4,5,8,9,12,13]].max(1); right=C[:,[2,3,6,7,10,11,14,15]].max(1)
print('left/right split', (left+right).sum())
# 8 subs of 8x4 (two horizontally adjacent 4x4 subs merged): sub index r4*2 + c4//2
rel84=np.zeros((len(g),8),bool)
rel48=np.zeros((len(g),8),bool)
for r4 in range(4):
    for c2 in range(2):
        rel84[:,r4*2+c2]=rel[:,4*r4+2*c2]|rel[:,4*r4+2*c2+1]
for r2_ in range(2):
    for c4 in range(4):
        rel48[:,r2_*4+c4]=rel[:,4*(2*r2_)+c4]|rel[:,4*(2*r2_+1)+c4]
for name,RR in (('8x4',rel84),('4x8',rel48)):
    C8=np.zeros((len(uk),8),np.int64)
    for s_ in range(8): C8[:,s_]=np.bincount(inv,weights=RR[:,s_],minlength=len(uk))
    print(name,'sum max8',C8.max(1).sum(),'cost (190/step)',C8.max(1).sum()*190/1e6)

# Cumulative (carry-over) walk: each group walks its whole tile list without per-batch lockstep;
# a warp's step count is then the max over its groups of the group's TOTAL relevant entries.
tb = uk // 100000  # tile of each (tile, batch) row
for name, cols in (('top', slice(0, 8)), ('bot', slice(8, 16))):
    pass
tot_top = np.zeros(T, np.int64); tot_bot = np.zeros(T, np.int64)
G = np.zeros((T, 16), np.int64)
np.add.at(G, tb, C)
cum = G[:, :8].max(1).sum() + G[:, 8:].max(1).sum()
print('lockstep per batch', (top + bot).sum(), 'cumulative per tile', cum,
      'ideal (mean)', C.sum() / 8)

# lockstep window size: steps = sum over (tile, window) of the max over a warp's 8 groups
for Wn in (32, 64, 96, 128, 256):
    bw = (m[tile] - 1 - pos) // Wn
    key2 = tile * 100000 + bw
    uk2, inv2 = np.unique(key2, return_inverse=True)
    C2 = np.zeros((len(uk2), 16), np.int64)
    for s_ in range(16): C2[:, s_] = np.bincount(inv2, weights=rel[:, s_], minlength=len(uk2))
    print('window', Wn, 'lockstep steps', C2[:, :8].max(1).sum() + C2[:, 8:].max(1).sum(),
          'windows', len(uk2))

# Entries past a sub-quarter's own last contributor (j >= max np over its 16 pixels) contribute
# exact zeros: lists that skip them (batch 128 lockstep)
sqmax = npr_p.reshape(ty_n, 4, 4, tx_n, 4, 4).max(axis=(2, 5))  # [ty, r4, tx, c4]
G16 = np.zeros((len(g), 16), np.int64)
for r4 in range(4):
    for c4 in range(4):
        G16[:, 4 * r4 + c4] = sqmax[ty, r4, tx, c4]
relx = rel & (pos[:, None] < G16)
print('relevant pairs', rel.sum(), 'before own max np', relx.sum())
for Wn in (128,):
    bw = (m[tile] - 1 - pos) // Wn
    key2 = tile * 100000 + bw
    uk2, inv2 = np.unique(key2, return_inverse=True)
    for nm, RR in (('all', rel), ('trimmed', relx)):
        C2 = np.zeros((len(uk2), 16), np.int64)
        for s_ in range(16): C2[:, s_] = np.bincount(inv2, weights=RR[:, s_], minlength=len(uk2))
        print(nm, 'window', Wn, 'lockstep steps', C2[:, :8].max(1).sum() + C2[:, 8:].max(1).sum())

# 2-lane groups over 4x2 half sub-quarters (16 groups per warp): finer culling, 2-lane reduce,
# lockstep over 16 lists per warp.  rel8[:, 2*s + h]: sub-quarter s, half h (top/bottom 2 rows)
rel8 = np.zeros((len(g), 32), bool)
for r4 in range(4):
    for c4 in range(4):
        for h in range(2):
            y0 = ty * 16 + 4 * r4 + 2 * h + 0.5; y1 = np.minimum(ty * 16 + 4 * r4 + 2 * h + 2, H) - 1 + 0.5
            dy = np.clip(v[g], y0, y1) - v[g]
            x0 = tx * 16 + 4 * c4 + 0.5; x1 = np.minimum(tx * 16 + 4 * c4 + 4, W) - 1 + 0.5
            dx = np.clip(u[g], x0, x1) - u[g]
            rel8[:, 2 * (4 * r4 + c4) + h] = (dx * dx + dy * dy <= r2m[g]) & (ty * 16 + 4 * r4 + 2 * h < H) & (tx * 16 + 4 * c4 < W)
bw = (m[tile] - 1 - pos) // 128
key2 = tile * 100000 + bw
uk2, inv2 = np.unique(key2, return_inverse=True)
C32 = np.zeros((len(uk2), 32), np.int64)
for s_ in range(32): C32[:, s_] = np.bincount(inv2, weights=rel8[:, s_], minlength=len(uk2))
steps8 = C32[:, :16].max(1).sum() + C32[:, 16:].max(1).sum()
print('4x2 groups: relevant group-entry pairs', rel8.sum(), '(x8 px =', rel8.sum() * 8, 'slots) vs 4x4', rel.sum() * 16,
      '; lockstep warp steps', steps8, '(x 16 groups x 8 px =', steps8 * 128, 'slots)')
