// Adaptive control of the isotropic 3D splat set: prune, merge, split as
// GPU compaction and append.  Control flow of adaptive_control
// (/root/reference/proj/src/optimize.cpp:221-284), rules for 3D splats as restated in the
// oracle (oracle/isg_oracle.c, or_adaptive_control dims == 3):
//
//   prune   keep splats with opacity >= eps; if none survives keep the first of maximal
//           opacity (prune_impl :153-174)                       -> stable compaction
//   merge   every pair with |mu_i - mu_j| < gamma min(sigma) and max colour difference < tol
//           qualifies (:232-244); pairs are taken greedily nearest-first on (dist, i, j), one
//           merge per splat (:246-259)
//             pair search: multi-level hash grid — splat i lives on level L_i, the smallest
//             L >= 0 with h0 2^L >= gamma sigma_i (h0 = gamma min sigma), in cell
//             floor(mu / (h0 2^L)); a pair is found once, from its smaller (sigma, index)
//             endpoint, by probing the <= 8 cells its gamma-sigma ball overlaps on every
//             occupied level >= L_i (the partner's level is >= L_i and its cell side >= the
//             ball radius)
//             matching: rounds of "locally dominant" edges — an edge is accepted when it is the
//             (dist, i, j)-minimum among live edges at both endpoints; this is exactly the
//             sequential greedy matching, in O(log) rounds
//             apply: merged splat replaces the lower index, the higher is dropped (a refused
//             merge still consumes both)              -> stable compaction
//   split   splats with sigma > split_sigma_max, widest first (ties: higher index first), while
//           the count stays <= max_particles (:263-281); the child replaces the parent in place
//           (mu + d sigma/2) and its twin is appended (mu - d sigma/2)
// Merge/split arithmetic is FP64 (this file is compiled with -fmad=false so every product and
// sum rounds like the oracle's) and rounded to FP32 once; directions come from Marsaglia's
// method on a splitmix64 stream keyed by (seed, round, parent index) — no transcendentals —
// so results are bit-identical to the oracle.
#include <algorithm>
#include <cmath>
#include <vector>

#include "isg_internal.cuh"

namespace isg {

namespace {

constexpr int kT = 256;

__device__ __forceinline__ uint64_t splitmix(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ void split_direction(uint64_t seed, uint64_t round, uint64_t index, double d[3]) {
  uint64_t s = seed ^ (round * 0xD1B54A32D192ED03ull) ^ (index * 0xA24BAED4963EE407ull);
  for (;;) {
    const double u1 = (double)(splitmix(s) >> 11) * 0x1.0p-52 - 1.0;
    const double u2 = (double)(splitmix(s) >> 11) * 0x1.0p-52 - 1.0;
    const double q = u1 * u1 + u2 * u2;
    if (q >= 1.0 || q == 0.0) continue;
    const double f = 2.0 * sqrt(1.0 - q);
    d[0] = u1 * f;
    d[1] = u2 * f;
    d[2] = 1.0 - 2.0 * q;
    return;
  }
}

// ---- stable compaction (block count -> block scan -> scatter) -----------------------------
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  uint32_t pre = 0, tot = 0;
  for (int i = 0; i < kT / 32; ++i) {
    pre += (i < w) ? s_warp[i] : 0u;
    tot += s_warp[i];
  }
  total = tot;
  __syncthreads();
  return pre + x - v;
}

__global__ void k_block_count(const uint8_t* __restrict__ flag, int64_t n, uint32_t* __restrict__ cnt) {
  __shared__ uint32_t s_warp[kT / 32];
  const int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x;
  uint32_t tot;
  block_excl_scan(i < n && flag[i] ? 1u : 0u, s_warp, tot);
  if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

// exclusive scan of nb block counts in one CTA; total -> *out_total
__global__ void k_scan_counts(uint32_t* __restrict__ cnt, int64_t nb, uint32_t* __restrict__ out_total) {
  __shared__ uint32_t s_warp[kT / 32];
  uint32_t carry = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += kT) {
    const int64_t b = b0 + threadIdx.x;
    const uint32_t v = b < nb ? cnt[b] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan(v, s_warp, tot);
    if (b < nb) cnt[b] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *out_total = carry;
}

// dst position of every kept item (reverse: positions counted from the end, i.e. the kept items
// land in descending index order)
__global__ void k_compact_pos(const uint8_t* __restrict__ flag, int64_t n,
                              const uint32_t* __restrict__ boff, const uint32_t* __restrict__ total,
                              bool reverse, uint32_t* __restrict__ pos) {
  __shared__ uint32_t s_warp[kT / 32];
  const int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x;
  const bool f = i < n && flag[i];
  uint32_t tot;
  const uint32_t ex = block_excl_scan(f ? 1u : 0u, s_warp, tot);
  if (i < n) {
    const uint32_t p = boff[blockIdx.x] + ex;
    pos[i] = f ? (reverse ? *total - 1u - p : p) : 0xFFFFFFFFu;
  }
}

__global__ void k_gather_scene(const float4* __restrict__ ms, const float4* __restrict__ co, int64_t n,
                               const uint32_t* __restrict__ pos, float4* __restrict__ ms_out,
                               float4* __restrict__ co_out) {
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    const uint32_t p = pos[i];
    if (p != 0xFFFFFFFFu) {
      ms_out[p] = ms[i];
      co_out[p] = co[i];
    }
  }
}

// ---- prune -----------------------------------------------------------------------------------
__global__ void k_prune_flags(const float4* __restrict__ co, int64_t n, double eps,
                              uint8_t* __restrict__ keep, unsigned long long* __restrict__ best) {
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    const float o = co[i].w + 0.0f;  // -0 -> +0, so the bit pattern orders like the value
    keep[i] = (double)o >= eps ? 1 : 0;
    // first index of maximal opacity: max of (bits(o) << 32 | ~i); opacities are >= 0
    atomicMax(best, ((unsigned long long)__float_as_uint(o) << 32) | (0xFFFFFFFFu - (uint32_t)i));
  }
}

__global__ void k_keep_best(const unsigned long long* __restrict__ best, const uint32_t* total,
                            uint8_t* __restrict__ keep) {
  if (*total == 0) keep[0xFFFFFFFFu - (uint32_t)(*best & 0xFFFFFFFFu)] = 1;
}

// ---- pair search -----------------------------------------------------------------------------
__device__ __forceinline__ int level_of(double gs, double h0) {
  int L = 0;
  double s = h0;
  while (s < gs && L < 63) {
    s *= 2.0;
    ++L;
  }
  return L;
}

__device__ __forceinline__ uint32_t cell_key(int L, long long cx, long long cy, long long cz) {
  uint64_t h = (uint64_t)cx * 0x9E3779B97F4A7C15ull;
  h ^= (uint64_t)cy * 0xC2B2AE3D27D4EB4Full + (h >> 29);
  h ^= (uint64_t)cz * 0x165667B19E3779F9ull + (h >> 32);
  h ^= h >> 33;
  h *= 0xFF51AFD7ED558CCDull;
  h ^= h >> 33;
  return ((uint32_t)L << 26) | (uint32_t)(h & 0x3FFFFFFull);
}

__global__ void k_sigma_min(const float4* __restrict__ ms, int64_t n, uint32_t* __restrict__ smin) {
  uint32_t m = 0x7F800000u;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT)
    m = min(m, __float_as_uint(ms[i].w));
  for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMin(smin, m);
}

__global__ void k_cell_keys(const float4* __restrict__ ms, int64_t n, double gamma,
                            const uint32_t* __restrict__ smin, uint32_t* __restrict__ key,
                            unsigned long long* __restrict__ level_mask) {
  const double h0 = gamma * (double)__uint_as_float(*smin);
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    const float4 m = ms[i];
    const int L = level_of(gamma * (double)m.w, h0);
    const double s = ldexp(h0, L);
    key[i] = cell_key(L, (long long)floor((double)m.x / s), (long long)floor((double)m.y / s),
                      (long long)floor((double)m.z / s));
    atomicOr(level_mask, 1ull << L);
  }
}

// open-addressing table: cell key -> first sorted position of the cell's run
__global__ void k_cell_table(const uint32_t* __restrict__ skey, int64_t n, uint32_t* __restrict__ tkey,
                             uint32_t* __restrict__ tval, uint32_t mask) {
  for (int64_t p = (int64_t)blockIdx.x * kT + threadIdx.x; p < n; p += (int64_t)gridDim.x * kT) {
    const uint32_t k = skey[p];
    if (p > 0 && skey[p - 1] == k) continue;
    uint32_t slot = (k * 0x9E3779B1u) & mask;
    for (;;) {
      const uint32_t prev = atomicCAS(&tkey[slot], 0xFFFFFFFFu, k);
      if (prev == 0xFFFFFFFFu) {
        tval[slot] = (uint32_t)p;
        break;
      }
      slot = (slot + 1) & mask;
    }
  }
}

struct Edge {
  double dist;
  uint32_t lo, hi;
};

__global__ void k_find_pairs(const float4* __restrict__ ms, const float4* __restrict__ co, int64_t n,
                             double gamma, double ctol, const uint32_t* __restrict__ smin,
                             const unsigned long long* __restrict__ level_mask,
                             const uint32_t* __restrict__ skey, const uint32_t* __restrict__ sval,
                             const uint32_t* __restrict__ tkey, const uint32_t* __restrict__ tval,
                             uint32_t mask, Edge* __restrict__ edges, int64_t edge_cap,
                             unsigned long long* __restrict__ n_edges) {
  const double h0 = gamma * (double)__uint_as_float(*smin);
  const unsigned long long lm = *level_mask;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    const float4 mi = ms[i];
    const float4 ci = co[i];
    const double r0 = gamma * (double)mi.w;
    const int Li = level_of(r0, h0);
    const double r = r0 * (1.0 + 1e-9);  // probe box slightly wider than the exact ball
    for (int L = Li; L < 64; ++L) {
      if (!((lm >> L) & 1ull)) continue;
      const double s = ldexp(h0, L);
      const long long x0 = (long long)floor(((double)mi.x - r) / s), x1 = (long long)floor(((double)mi.x + r) / s);
      const long long y0 = (long long)floor(((double)mi.y - r) / s), y1 = (long long)floor(((double)mi.y + r) / s);
      const long long z0 = (long long)floor(((double)mi.z - r) / s), z1 = (long long)floor(((double)mi.z + r) / s);
      for (long long cx = x0; cx <= x1; ++cx)
        for (long long cy = y0; cy <= y1; ++cy)
          for (long long cz = z0; cz <= z1; ++cz) {
            const uint32_t k = cell_key(L, cx, cy, cz);
            uint32_t slot = (k * 0x9E3779B1u) & mask, start = 0xFFFFFFFFu;
            for (;;) {
              const uint32_t tk = tkey[slot];
              if (tk == k) {
                start = tval[slot];
                break;
              }
              if (tk == 0xFFFFFFFFu) break;
              slot = (slot + 1) & mask;
            }
            if (start == 0xFFFFFFFFu) continue;
            for (int64_t p = start; p < n && skey[p] == k; ++p) {
              const uint32_t j = sval[p];
              if (j == (uint32_t)i) continue;
              const float4 mj = ms[j];
              // the pair is found from its smaller (sigma, index) endpoint only
              if (!(mj.w > mi.w || (mj.w == mi.w && j > (uint32_t)i))) continue;
              // exact cell membership (hash collisions share runs)
              if (level_of(gamma * (double)mj.w, h0) != L) continue;
              if ((long long)floor((double)mj.x / s) != cx || (long long)floor((double)mj.y / s) != cy ||
                  (long long)floor((double)mj.z / s) != cz)
                continue;
              const uint32_t lo = min((uint32_t)i, j), hi = max((uint32_t)i, j);
              const float4 mlo = lo == (uint32_t)i ? mi : mj, mhi = lo == (uint32_t)i ? mj : mi;
              const double dx = (double)mlo.x - (double)mhi.x, dy = (double)mlo.y - (double)mhi.y,
                           dz = (double)mlo.z - (double)mhi.z;
              double ss = 0.0;
              ss = ss + dx * dx;
              ss = ss + dy * dy;
              ss = ss + dz * dz;
              const double dist = sqrt(ss);
              if (dist >= gamma * (double)fminf(mi.w, mj.w)) continue;
              const float4 cj = co[j];
              const float4 clo = lo == (uint32_t)i ? ci : cj, chi = lo == (uint32_t)i ? cj : ci;
              double cd = 0.0;
              cd = fmax(cd, fabs((double)clo.x - (double)chi.x));
              cd = fmax(cd, fabs((double)clo.y - (double)chi.y));
              cd = fmax(cd, fabs((double)clo.z - (double)chi.z));
              if (cd >= ctol) continue;
              const unsigned long long e = atomicAdd(n_edges, 1ull);
              if ((int64_t)e < edge_cap) edges[e] = Edge{dist, lo, hi};
            }
          }
    }
  }
}

// ---- greedy matching in locally-dominant rounds -------------------------------------------------
__device__ __forceinline__ bool edge_live(const Edge& e, const uint8_t* matched) {
  return !matched[e.lo] && !matched[e.hi];
}

__global__ void k_match_min_d(const Edge* __restrict__ edges, int64_t ne, const uint8_t* __restrict__ matched,
                              unsigned long long* __restrict__ bestd) {
  for (int64_t k = (int64_t)blockIdx.x * kT + threadIdx.x; k < ne; k += (int64_t)gridDim.x * kT) {
    const Edge e = edges[k];
    if (!edge_live(e, matched)) continue;
    const unsigned long long d = (unsigned long long)__double_as_longlong(e.dist);
    atomicMin(&bestd[e.lo], d);
    atomicMin(&bestd[e.hi], d);
  }
}

__global__ void k_match_min_ij(const Edge* __restrict__ edges, int64_t ne, const uint8_t* __restrict__ matched,
                               const unsigned long long* __restrict__ bestd,
                               unsigned long long* __restrict__ bestij) {
  for (int64_t k = (int64_t)blockIdx.x * kT + threadIdx.x; k < ne; k += (int64_t)gridDim.x * kT) {
    const Edge e = edges[k];
    if (!edge_live(e, matched)) continue;
    const unsigned long long d = (unsigned long long)__double_as_longlong(e.dist);
    const unsigned long long ij = ((unsigned long long)e.lo << 32) | e.hi;
    if (bestd[e.lo] == d) atomicMin(&bestij[e.lo], ij);
    if (bestd[e.hi] == d) atomicMin(&bestij[e.hi], ij);
  }
}

__global__ void k_match_accept(const Edge* __restrict__ edges, int64_t ne, uint8_t* __restrict__ matched,
                               const unsigned long long* __restrict__ bestd,
                               const unsigned long long* __restrict__ bestij,
                               uint32_t* __restrict__ partner, unsigned int* __restrict__ accepted) {
  for (int64_t k = (int64_t)blockIdx.x * kT + threadIdx.x; k < ne; k += (int64_t)gridDim.x * kT) {
    const Edge e = edges[k];
    if (!edge_live(e, matched)) continue;
    const unsigned long long d = (unsigned long long)__double_as_longlong(e.dist);
    const unsigned long long ij = ((unsigned long long)e.lo << 32) | e.hi;
    if (bestd[e.lo] == d && bestd[e.hi] == d && bestij[e.lo] == ij && bestij[e.hi] == ij) {
      partner[e.lo] = e.hi;
      partner[e.hi] = e.lo;
      atomicAdd(accepted, 1u);
    }
  }
}

// commit the round's accepted edges (after every edge was tested against the old state)
__global__ void k_match_commit(int64_t n, const uint32_t* __restrict__ partner, uint8_t* __restrict__ matched) {
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT)
    if (partner[i] != 0xFFFFFFFFu) matched[i] = 1;
}

// merge (oracle or_merge, dims 3): lower index receives the merged splat, higher is dropped
__global__ void k_apply_merge(float4* __restrict__ ms, float4* __restrict__ co, int64_t n,
                              const uint32_t* __restrict__ partner, uint8_t* __restrict__ keep,
                              unsigned int* __restrict__ merged) {
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    const uint32_t j = partner[i];
    if (j == 0xFFFFFFFFu || j < (uint32_t)i) continue;
    const float4 a = ms[i], b = ms[j], ca = co[i], cb = co[j];
    const double s1 = a.w, s2 = b.w;
    const double w1 = (double)ca.w * (s1 * s1), w2 = (double)cb.w * (s2 * s2);
    const double total = w1 + w2;
    if (fabs(total) < 1e-12) continue;
    const double mx = (w1 * (double)a.x + w2 * (double)b.x) / total;
    const double my = (w1 * (double)a.y + w2 * (double)b.y) / total;
    const double mz = (w1 * (double)a.z + w2 * (double)b.z) / total;
    const double q = (w1 * (s1 * s1) + w2 * (s2 * s2)) / total;
    if (!(q > 0.0) || !isfinite(q) || !isfinite(mx) || !isfinite(my) || !isfinite(mz)) continue;
    const float sg = (float)sqrt(q);
    if (!(sg > 0.0f)) continue;
    const double o = total / q;
    ms[i] = make_float4((float)mx, (float)my, (float)mz, sg);
    co[i] = make_float4((float)((w1 * (double)ca.x + w2 * (double)cb.x) / total),
                        (float)((w1 * (double)ca.y + w2 * (double)cb.y) / total),
                        (float)((w1 * (double)ca.z + w2 * (double)cb.z) / total),
                        (float)(o < 1.0 ? o : 1.0));
    keep[j] = 0;
    atomicAdd(merged, 1u);
  }
}

// ---- split -------------------------------------------------------------------------------------
__global__ void k_split_flags(const float4* __restrict__ ms, int64_t n, double smax,
                              uint8_t* __restrict__ cand, uint32_t* __restrict__ key) {
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    const float s = ms[i].w;
    cand[i] = (double)s > smax ? 1 : 0;
    key[i] = ~__float_as_uint(s);  // ascending key = descending sigma (sigma > 0)
  }
}

__global__ void k_split_list(const uint8_t* __restrict__ cand, const uint32_t* __restrict__ key,
                             const uint32_t* __restrict__ pos, int64_t n, uint32_t* __restrict__ ckey,
                             uint32_t* __restrict__ cidx) {
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT)
    if (cand[i]) {
      ckey[pos[i]] = key[i];
      cidx[pos[i]] = (uint32_t)i;
    }
}

__global__ void k_apply_split(float4* __restrict__ ms, float4* __restrict__ co, int64_t count,
                              const uint32_t* __restrict__ parent, int64_t k_split, uint64_t seed,
                              uint64_t round) {
  for (int64_t r = (int64_t)blockIdx.x * kT + threadIdx.x; r < k_split; r += (int64_t)gridDim.x * kT) {
    const uint32_t i = parent[r];
    const float4 p = ms[i];
    double d[3];
    split_direction(seed, round, i, d);
    const double h = 0.5 * (double)p.w;
    const double ox = h * d[0], oy = h * d[1], oz = h * d[2];
    const float sg = (float)((double)p.w * sqrt(0.5));
    ms[count + r] = make_float4((float)((double)p.x - ox), (float)((double)p.y - oy),
                                (float)((double)p.z - oz), sg);
    co[count + r] = co[i];
    ms[i] = make_float4((float)((double)p.x + ox), (float)((double)p.y + oy),
                        (float)((double)p.z + oz), sg);
  }
}

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, 148 * 16)); }

}  // namespace

// Stable compaction helper: pos[i] = destination of item i (or ~0), returns the kept count
// (synchronises).  scratch: >= ceil(n / 256) + 1 words.
static cudaError_t compact_positions(const uint8_t* flag, int64_t n, bool reverse, uint32_t* pos,
                                     uint32_t* scratch, uint32_t* h_total, cudaStream_t st) {
  const int64_t nb = (n + kT - 1) / kT;
  if (nb == 0) {
    *h_total = 0;
    return cudaSuccess;
  }
  k_block_count<<<(unsigned)nb, kT, 0, st>>>(flag, n, scratch);
  k_scan_counts<<<1, kT, 0, st>>>(scratch, nb, scratch + nb);
  k_compact_pos<<<(unsigned)nb, kT, 0, st>>>(flag, n, scratch, scratch + nb, reverse, pos);
  cudaMemcpyAsync(h_total, scratch + nb, sizeof(uint32_t), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  return cudaGetLastError();
}

struct AdaptScratch {
  int64_t n_cap = 0, alloc_cap = 0, edge_cap = 0;
  uint32_t t_cap = 0;
  uint8_t* flag = nullptr;
  uint32_t *pos = nullptr, *scratch = nullptr, *partner = nullptr, *tk = nullptr, *tv = nullptr;
  unsigned long long *best = nullptr, *bestd = nullptr, *bestij = nullptr;
  unsigned int* acc = nullptr;
  void* edges = nullptr;  // Edge[edge_cap]
  float4 *ms_tmp = nullptr, *co_tmp = nullptr;
  uint32_t* h = nullptr;  // pinned
};

void adapt_scratch_free(AdaptScratch* s) {
  if (!s) return;
  cudaFree(s->flag);
  cudaFree(s->pos);
  cudaFree(s->scratch);
  cudaFree(s->partner);
  cudaFree(s->tk);
  cudaFree(s->tv);
  cudaFree(s->best);
  cudaFree(s->bestd);
  cudaFree(s->bestij);
  cudaFree(s->acc);
  cudaFree(s->edges);
  cudaFree(s->ms_tmp);
  cudaFree(s->co_tmp);
  cudaFreeHost(s->h);
  delete s;
}

template <class T>
static cudaError_t regrow(T*& p, size_t count) {
  cudaFree(p);
  p = nullptr;
  return cudaMalloc(&p, count * sizeof(T));
}

cudaError_t adaptive_control(float4*& ms, float4*& co, int64_t n, int64_t n_alloc,
                             const AdaptParamsDev& p, uint64_t seed, uint64_t round,
                             SortScratch& sort, uint32_t* keys[2], uint32_t* vals[2],
                             AdaptScratch*& S, AdaptCounts* counts, cudaStream_t st,
                             int64_t* launches) {
  cudaError_t err = cudaSuccess;
  counts->n_before = n;
  counts->n_pruned = counts->n_merged = counts->n_split = 0;
  counts->n_after = n;
  if (n == 0) return cudaSuccess;
#define ADAPT_CHECK(x)        \
  do {                        \
    err = (x);                \
    if (err != cudaSuccess) { \
      return err;             \
    }                         \
  } while (0)
  if (!S) S = new AdaptScratch();
  const int64_t nb = (n + kT - 1) / kT;
  if (!S->h) ADAPT_CHECK(cudaMallocHost(&S->h, 16 * sizeof(uint32_t)));
  if (!S->best) {
    ADAPT_CHECK(cudaMalloc(&S->best, 4 * sizeof(unsigned long long)));
    ADAPT_CHECK(cudaMalloc(&S->acc, 4 * sizeof(unsigned int)));
  }
  if (n > S->n_cap) {
    ADAPT_CHECK(regrow(S->flag, n));
    ADAPT_CHECK(regrow(S->pos, n));
    ADAPT_CHECK(regrow(S->scratch, nb + 8));
    ADAPT_CHECK(regrow(S->partner, n));
    ADAPT_CHECK(regrow(S->bestd, n));
    ADAPT_CHECK(regrow(S->bestij, n));
    S->n_cap = n;
  }
  if (n_alloc > S->alloc_cap) {
    ADAPT_CHECK(regrow(S->ms_tmp, n_alloc));
    ADAPT_CHECK(regrow(S->co_tmp, n_alloc));
    S->alloc_cap = n_alloc;
  }
  uint8_t* flag = S->flag;
  uint32_t *pos = S->pos, *scratch = S->scratch, *partner = S->partner;
  unsigned long long *best = S->best, *bestd = S->bestd, *bestij = S->bestij;
  unsigned int* acc = S->acc;
  uint32_t* h = S->h;
  float4 *ms_tmp = S->ms_tmp, *co_tmp = S->co_tmp;
  const int g = grid_for(n);

  // ---- prune --------------------------------------------------------------------------------
  cudaMemsetAsync(best, 0, 4 * sizeof(unsigned long long), st);
  k_prune_flags<<<g, kT, 0, st>>>(co, n, p.prune_threshold, flag, best);
  ADAPT_CHECK(compact_positions(flag, n, false, pos, scratch, h, st));
  if (h[0] == 0) {
    k_keep_best<<<1, 1, 0, st>>>(best, scratch + nb, flag);
    ADAPT_CHECK(compact_positions(flag, n, false, pos, scratch, h, st));
  }
  int64_t m = h[0];
  k_gather_scene<<<g, kT, 0, st>>>(ms, co, n, pos, ms_tmp, co_tmp);
  std::swap(ms, ms_tmp);
  std::swap(co, co_tmp);
  S->ms_tmp = ms_tmp;  // the scene's previous buffers become the scratch
  S->co_tmp = co_tmp;
  counts->n_pruned = n - m;
  *launches += 6;

  // ---- merge: pairs ---------------------------------------------------------------------------
  uint32_t* smin = scratch + nb + 2;
  unsigned long long* lmask = best + 1;
  cudaMemsetAsync(smin, 0x7F, sizeof(uint32_t), st);
  cudaMemsetAsync(lmask, 0, sizeof(unsigned long long), st);
  const int gm = grid_for(m);
  k_sigma_min<<<gm, kT, 0, st>>>(ms, m, smin);
  k_cell_keys<<<gm, kT, 0, st>>>(ms, m, p.merge_distance_factor, smin, keys[0], lmask);
  *h = (uint32_t)m;
  uint32_t* n_dev = scratch + nb + 3;
  cudaMemcpyAsync(n_dev, h, sizeof(uint32_t), cudaMemcpyHostToDevice, st);
  const int sb = radix_sort_pairs(keys, vals, true, n_dev, m, 32, sort, st, launches);
  uint32_t tsize = 1;
  while (tsize < 2 * (uint64_t)m) tsize <<= 1;
  if (tsize > S->t_cap) {
    ADAPT_CHECK(regrow(S->tk, tsize));
    ADAPT_CHECK(regrow(S->tv, tsize));
    S->t_cap = tsize;
  }
  uint32_t *tk = S->tk, *tv = S->tv;
  cudaMemsetAsync(tk, 0xFF, tsize * sizeof(uint32_t), st);
  k_cell_table<<<gm, kT, 0, st>>>(keys[sb], m, tk, tv, tsize - 1);
  int64_t edge_cap = std::max<int64_t>(S->edge_cap, std::max<int64_t>(4 * m, 1024));
  int64_t ne = 0;
  unsigned long long* n_edges = best + 2;
  Edge* edges = static_cast<Edge*>(S->edges);
  for (int attempt = 0; attempt < 4; ++attempt) {
    if (edge_cap > S->edge_cap) {
      ADAPT_CHECK(regrow(edges, edge_cap));
      S->edges = edges;
      S->edge_cap = edge_cap;
    }
    cudaMemsetAsync(n_edges, 0, sizeof(unsigned long long), st);
    k_find_pairs<<<gm, kT, 0, st>>>(ms, co, m, p.merge_distance_factor, p.merge_color_tol, smin,
                                    lmask, keys[sb], vals[sb], tk, tv, tsize - 1, edges, edge_cap,
                                    n_edges);
    unsigned long long ne_h = 0;
    cudaMemcpyAsync(&ne_h, n_edges, sizeof(ne_h), cudaMemcpyDeviceToHost, st);
    ADAPT_CHECK(cudaStreamSynchronize(st));
    ADAPT_CHECK(cudaGetLastError());
    ne = (int64_t)ne_h;
    if (ne <= edge_cap) break;
    edge_cap = ne + ne / 4 + 1024;
  }
  *launches += 5;

  // ---- merge: greedy matching ----------------------------------------------------------------
  cudaMemsetAsync(flag, 0, m, st);  // matched
  cudaMemsetAsync(partner, 0xFF, m * sizeof(uint32_t), st);
  if (ne > 0) {
    const int ge = grid_for(ne);
    for (;;) {
      cudaMemsetAsync(bestd, 0xFF, m * sizeof(unsigned long long), st);
      cudaMemsetAsync(bestij, 0xFF, m * sizeof(unsigned long long), st);
      cudaMemsetAsync(acc, 0, sizeof(unsigned int), st);
      k_match_min_d<<<ge, kT, 0, st>>>(edges, ne, flag, bestd);
      k_match_min_ij<<<ge, kT, 0, st>>>(edges, ne, flag, bestd, bestij);
      k_match_accept<<<ge, kT, 0, st>>>(edges, ne, flag, bestd, bestij, partner, acc);
      k_match_commit<<<gm, kT, 0, st>>>(m, partner, flag);
      *launches += 4;
      unsigned int a_h = 0;
      cudaMemcpyAsync(&a_h, acc, sizeof(a_h), cudaMemcpyDeviceToHost, st);
      ADAPT_CHECK(cudaStreamSynchronize(st));
      if (a_h == 0) break;
    }
  }
  // apply merges; keep = 1 except merged-away partners
  cudaMemsetAsync(flag, 1, m, st);
  cudaMemsetAsync(acc + 1, 0, sizeof(unsigned int), st);
  k_apply_merge<<<gm, kT, 0, st>>>(ms, co, m, partner, flag, acc + 1);
  ADAPT_CHECK(compact_positions(flag, m, false, pos, scratch, h, st));
  const int64_t c = h[0];
  k_gather_scene<<<gm, kT, 0, st>>>(ms, co, m, pos, ms_tmp, co_tmp);
  std::swap(ms, ms_tmp);
  std::swap(co, co_tmp);
  S->ms_tmp = ms_tmp;
  S->co_tmp = co_tmp;
  counts->n_merged = m - c;
  *launches += 5;

  // ---- split ---------------------------------------------------------------------------------
  int64_t count = c;
  const int64_t budget = std::max<int64_t>(0, p.max_particles - c);
  if (budget > 0 && c > 0) {
    const int gc = grid_for(c);
    k_split_flags<<<gc, kT, 0, st>>>(ms, c, p.split_sigma_max, flag, keys[0]);
    ADAPT_CHECK(compact_positions(flag, c, true, pos, scratch, h, st));  // descending index
    const int64_t nc = h[0];
    *launches += 4;
    if (nc > 0) {
      k_split_list<<<gc, kT, 0, st>>>(flag, keys[0], pos, c, keys[1], vals[1]);
      // stable sort of the (descending-index) candidates by descending sigma
      uint32_t* k2[2] = {keys[1], keys[0]};
      uint32_t* v2[2] = {vals[1], vals[0]};
      *h = (uint32_t)nc;
      cudaMemcpyAsync(n_dev, h, sizeof(uint32_t), cudaMemcpyHostToDevice, st);
      const int cb = radix_sort_pairs(k2, v2, false, n_dev, nc, 32, sort, st, launches);
      const int64_t ks = std::min(nc, budget);
      k_apply_split<<<grid_for(ks), kT, 0, st>>>(ms, co, c, v2[cb], ks, seed, round);
      count = c + ks;
      counts->n_split = ks;
      *launches += 2;
    }
  }
  ADAPT_CHECK(cudaStreamSynchronize(st));
  ADAPT_CHECK(cudaGetLastError());
  counts->n_after = count;
#undef ADAPT_CHECK
  return cudaSuccess;
}

}  // namespace isg
