// Latency kernel family: one ligand is spread over the whole GPU.
//
//  k_align_latency    (ds_align.cu)  blocks = ligand x restart x atom chunk, lane = ax
//  k_optimize_latency (this file)    one CTA per (ligand, restart) — the paper's "grid level =
//                                    initial poses" — with every thread of the
//                                    CTA on each step of a fragment; the CTA barrier is the paper's
//                                    block-level synchronisation.  Per fragment
//                                    five barrier-separated phases, all 256 threads busy in each:
//                                    (A) per-warp ballots of M / C' over 32-atom slots + the base
//                                    score + the axis, (B) compaction + cylindrical coordinates,
//                                    (C) flat (moving, complement) candidate test, (D) the angle
//                                    sweep, (E) best angle (every warp, redundantly) + commit.
//                                    Each CTA rescores its own final pose (speculatively, so the
//                                    rescore runs on N SMs at once); the last CTA of a ligand to
//                                    finish runs select_poses and picks the best kept pose
//                                    (PAPER.md:344-348).
// Numeric recipe identical to the batched family: results are bit-identical.
#include <cooperative_groups.h>
#include <limits.h>
#include <stdio.h>
#include <stdlib.h>

#include <map>
#include <mutex>

#include "ds_kernels.cuh"

namespace cg = cooperative_groups;

namespace ds {

#ifndef DS_LAT_THREADS
#define DS_LAT_THREADS 256
#endif
constexpr int kLatThreads = DS_LAT_THREADS;
constexpr int kLatWarps = kLatThreads / 32;
static_assert(kLatThreads >= DS_MAX_ATOMS, "phase (A) gives every atom its own thread");
constexpr int kLatChunk = 8;

struct LatRec {  // per (ligand, restart), read by the ligand's last CTA
  int geom, valid, degen, align_score;
  int degen_f;     // the fragment a DegenerateAxis stopped this restart at
  unsigned evals, pairs, exits, rot;
  long long chem;  // rescore of the restart's final pose (P11), valid poses only
};

constexpr int kLatCand = 8;

// state of the per-restart tail (final pose, rescore, record; the ligand's last CTA: select)
struct LatTail {
  int is_last;
  int geom;
  int ord[DS_MAX_RESTARTS], kept[DS_MAX_RESTARTS], nkept;
  unsigned dis[DS_MAX_RESTARTS];
  unsigned long long chem;
  int heavy;
  unsigned s_cnt[4], s_nal;
  int s_degf;
  LatRec rec[DS_MAX_RESTARTS];  // the ligand's per-restart records, staged by the last CTA
  int nvp;                      // valid restarts
  uint16_t vp[DS_MAX_RESTARTS * (DS_MAX_RESTARTS - 1) / 2];  // restart pairs as p | q << 8
};

struct LatSmem {
  float4 u[DS_MAX_ATOMS];
  float2 chr[DS_MAX_ATOMS];     // cylindrical (h, r) of the C' atoms
  float2 chm[DS_MAX_ATOMS];     // ... and of the moving atoms
  uint8_t mlist[DS_MAX_ATOMS];
  uint8_t clist[DS_MAX_ATOMS];
  uint8_t cl[DS_MAX_ATOMS][kLatCand];  // bump candidates (atom indices) per moving atom
  unsigned cn[DS_MAX_ATOMS];           // their count (> kLatCand: scan all of C')
  int ascore[32];
  int bcode[32];                // early exit: the smallest bumping moving slot per angle (P14 rows)
  unsigned abump;
  unsigned key;
  int degen, degen_f;
  unsigned pairs;
  LatTail t;
};

// dynamic shared memory: [trig 360][fragment records][weights][bin LUT][grid (if it fits)]
__host__ __device__ inline size_t lat_w_bytes(int nb) { return ((size_t)DS_N_TYPES * DS_N_TYPES * (nb + 1) * 4 + 15) & ~(size_t)15; }
__host__ __device__ inline size_t lat_lut_bytes(int lut_cap) { return ((size_t)(lut_cap + 1) + 15) & ~(size_t)15; }
__host__ __device__ inline size_t lat_base_bytes(int nb, int lut_cap) {
  return 360 * sizeof(float2) + 2 * (DS_MAX_ATOMS - 2) * sizeof(uint4) + lat_w_bytes(nb) + lat_lut_bytes(lut_cap);
}

// exact rescore bin (P11): the pocket's LUT (staged in shared memory) when it has one, else the compares
__device__ __forceinline__ int lat_bin(const PocketView &pk, const uint8_t *slut, float d2) {
  if (pk.lut_cap >= 0) return slut[min((unsigned)__float_as_int(d2) >> pk.lut_shift, (unsigned)pk.lut_cap)];
  int b = 0;
  for (int q = 0; q < pk.nb; ++q) b += !(d2 < pk.ub2[q]);
  return b;
}

// grid lookup: the CTA's shared-memory copy when the pocket fits, else the L2-resident global copy
template <bool kSmemGrid>
__device__ __forceinline__ int lat_grid_val(const uint8_t *grid, int idx) {
  return (kSmemGrid ? (int)grid[idx] : (int)__ldg(grid + idx)) - 128;
}

__device__ __forceinline__ float2 lat_cyl(float4 p, float3 a, float kx, float ky, float kz) {
  const float wx = p.x - a.x, wy = p.y - a.y, wz = p.z - a.z;
  const float h = wx * kx + wy * ky + wz * kz;
  return make_float2(h, sqrtf(fmaxf(wx * wx + wy * wy + wz * wz - h * h, 0.f)));
}

__device__ __forceinline__ float3 lat_torsion_pos(const float2 *trig, int step_t, int k, float kx, float ky, float kz,
                                                  float3 a, float4 p) {
  if (k == 0) return make_float3(p.x, p.y, p.z);
  const float2 cs = trig[k * step_t];
  float R[9];
  torsion_matrix(kx, ky, kz, cs.x, cs.y, R);
  return torsion_apply(R, a, p.x, p.y, p.z);
}

// exact n / d for 0 <= n <= 2^16, 1 <= d <= 2^16: float estimate, then a one-step correction
__device__ __forceinline__ int small_div(int n, int d) {
  int q = (int)__fmul_rn((float)n, __frcp_rn((float)d));
  const int r = n - q * d;
  q += (r >= d) - (r < 0);
  return q;
}

// nearest bump candidate of moving atom m at its rotated position q (the cylindrical candidates,
// or all of C' when they overflowed the list)
__device__ __forceinline__ float lat_min_d2(const LatSmem &S, int m, int nC, float3 q) {
  float mind = __int_as_float(0x7f800000);
  const unsigned cnt = S.cn[m];
  if (cnt <= (unsigned)kLatCand) {
    for (unsigned t = 0; t < cnt; ++t) {
      const float4 y = S.u[S.cl[m][t]];
      mind = fminf(mind, dist2(q.x, q.y, q.z, y.x, y.y, y.z));
    }
  } else {
    for (int c = 0; c < nC; ++c) {
      const float4 y = S.u[S.clist[c]];
      mind = fminf(mind, dist2(q.x, q.y, q.z, y.x, y.y, y.z));
    }
  }
  return mind;
}

#ifdef DS_SPEC_PROBE
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ unsigned long long g_marks[64][8];
__device__ unsigned long long g_marks2[64][8];
#define MARK2(tag, id) \
  if (threadIdx.x == 0) g_marks2[(id) & 63][tag] = gtimer()
__device__ long long g_steps[16][16][8];  // spread kernel, cluster 0: [CTA][step][point] clock64 deltas
#define SPROBE(k) \
  if (blockIdx.x < kSpecH && (f >> 1) < 16) g_steps[lead ? kSpecH : blockIdx.x][f >> 1][k] = clock64() - t_step
#define MARK(tag, id) \
  if (threadIdx.x == 0) g_marks[(id) & 63][tag] = gtimer()
#else
#define MARK(tag, id)
#define MARK2(tag, id)
#define SPROBE(k)
#endif

// a slice of the rescore sum (P11) of the pose U by thread t of nth: with enough threads, one
// work unit (pocket atom j, chunk of <= 16 ligand atoms) each, else a pocket atom per thread
// (loaded once) over every chunk.  Each int32 partial holds at most part_terms terms, so it cannot
// overflow; the 64-bit total is exact, hence independent of the split.
__device__ __forceinline__ int lat_rescore_chunk(const float4 *U, int i0, int i1, float4 y, const int32_t *wcol, int nb1,
                                                 const PocketView &pk, const uint8_t *slut) {
  int part = 0;
#pragma unroll 4
  for (int i = i0; i < i1; ++i) {
    const float4 x = U[i];
    const float d2 = dist2(x.x, x.y, x.z, y.x, y.y, y.z);
    part += wcol[(int)x.w * DS_N_TYPES * nb1 + lat_bin(pk, slut, d2)];
  }
  return part;
}
__device__ __forceinline__ long long lat_rescore_acc(const float4 *U, int A, const PocketView &pk, const int32_t *sw,
                                                     const uint8_t *slut, int t, int nth) {
  const int nb1 = pk.nb + 1;
  const int CH = min(pk.part_terms, 16);
  const int nch = (A + CH - 1) / CH;
  long long acc = 0;
  if (pk.n_atoms * nch <= nth) {
    if (t < pk.n_atoms * nch) {
      const int j = t / nch, c = t - j * nch;
      const float4 y = __ldg(pk.patoms + j);
      acc = lat_rescore_chunk(U, c * CH, min(A, c * CH + CH), y, sw + (int)y.w * nb1, nb1, pk, slut);
    }
    return acc;
  }
  for (int j = t; j < pk.n_atoms; j += nth) {
    const float4 y = __ldg(pk.patoms + j);
    const int32_t *wcol = sw + (int)y.w * nb1;
    for (int i0 = 0; i0 < A; i0 += CH) acc += lat_rescore_chunk(U, i0, min(A, i0 + CH), y, wcol, nb1, pk, slut);
  }
  return acc;
}

// one atom's term of the RMSD sum (P12): (dx^2 + dy^2) + dz^2 in f64, 0 for a hydrogen
__device__ __forceinline__ double rmsd_term(float4 x, float4 y) {
  if (x.w == 0.f) return 0.0;
  const double dx = __dsub_rn((double)x.x, (double)y.x);
  const double dy = __dsub_rn((double)x.y, (double)y.y);
  const double dz = __dsub_rn((double)x.z, (double)y.z);
  double v = __dmul_rn(dx, dx);
  v = __dadd_rn(v, __dmul_rn(dy, dy));
  return __dadd_rn(v, __dmul_rn(dz, dz));
}

// the restart's tail, entered by every thread of the CTA with U final (after a barrier) and
// T.heavy = T.geom = T.chem = 0: final pose to the scratch, grid score, speculative rescore
// (P11; kRescore false: the caller has summed it into T.chem), the per-restart record; the
// ligand's last CTA to finish runs select_poses (P12) and writes the ligand's result
//
template <int NTH, bool kRescore>
__device__ __forceinline__ void lat_tail(LatTail &T, const float4 *U, int degen, int degen_f, int total, int valid,
                                         unsigned key, int ix, int iy, int rot, unsigned evals, unsigned pairs,
                                         unsigned exits, const PocketView &pk, const DockParams &dp, const int32_t *sw,
                                         const uint8_t *slut, const OptOut &out, LatRec *recs, int *done, int lig,
                                         int r, int a0, int A, int f0, int F, float4 *stage, int stage_bytes) {
  const int tid = threadIdx.x, lane = tid & 31;
  // ---- final pose, geometric score, per-restart record ----
  float4 *scr = out.final_u + ((size_t)lig * dp.N + r) * DS_MAX_ATOMS;
  if (!degen) {
    int hv = 0;
    for (int i = tid; i < A; i += NTH) {
      const float4 p = U[i];
      hv += p.w != 0.f;
      scr[i] = p;
    }
    hv = (int)__reduce_add_sync(kFull, (unsigned)hv);
    if (lane == 0) atomicAdd(&T.heavy, hv);
    if (tid == 0) T.geom = total;
  }
  __syncthreads();
  // ---- speculative rescore of this restart's pose (P11, exact fixed point): every CTA of the
  // ligand does its own in parallel, the last one only picks among the kept poses ----
  if (kRescore && !degen && valid) {
    long long acc = lat_rescore_acc(U, A, pk, sw, slut, tid, NTH);
    // warp sum then one shared 64-bit add per warp (two's complement: exact for signed sums)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if (lane == 0) atomicAdd(&T.chem, (unsigned long long)acc);
  }
  __syncthreads();
  MARK(3, lig * dp.N + r);
  if (tid == 0) {
    LatRec rec;
    rec.chem = (long long)T.chem;
    rec.geom = T.geom;
    rec.valid = valid;
    rec.degen = degen;
    rec.degen_f = degen ? degen_f : 0;
    rec.align_score = (int)(key >> 16) - 32768;
    rec.evals = evals;
    rec.pairs = pairs;
    rec.exits = exits;
    rec.rot = (unsigned)rot;
    recs[(size_t)lig * dp.N + r] = rec;
    if (out.rrec) {
      ds_restart_record rr;
      rr.align_score = rec.align_score;
      rr.final_geom = rec.geom;
      rr.ax = (uint8_t)ix;
      rr.ay = (uint8_t)iy;
      rr.valid = (uint8_t)valid;
      rr.kept = 0;
      rr.reserved = 0;
      out.rrec[(size_t)lig * dp.N + r] = rr;
    }
    __threadfence();  // release: this CTA's records and final pose before its count
    const bool last = atomicAdd(done + lig, 1) == dp.N - 1;
    if (last) {
      __threadfence();  // acquire: every other CTA's records and poses
      done[lig] = 0;    // every CTA of the ligand has counted in: reset for the next call
    }
    T.is_last = last;
  }
  __syncthreads();
  MARK2(0, lig * dp.N + r);
  if (!T.is_last) return;

  // ---- the ligand's last CTA: select_poses (P12), best rescored kept pose ----
  // one L2 round trip: every restart's record, and (when they fit the free grid region) every
  // restart's final pose and torsion indices
  const float4 *base_scr = out.final_u + (size_t)lig * dp.N * DS_MAX_ATOMS;
  const int N = dp.N, nst = N * A, nrt = F * N;
  const int npairs = N * (N - 1) / 2;
  const size_t pose_bytes = (size_t)nst * sizeof(float4), rt_bytes = ((size_t)nrt + 15) & ~(size_t)15;
  const bool posed = stage != nullptr && pose_bytes + rt_bytes <= (size_t)stage_bytes;
  uint8_t *srt = posed ? reinterpret_cast<uint8_t *>(stage + nst) : nullptr;
  {
    const unsigned *src = reinterpret_cast<const unsigned *>(recs + (size_t)lig * N);
    unsigned *dst = reinterpret_cast<unsigned *>(T.rec);
    for (int w = tid; w < N * (int)(sizeof(LatRec) / 4); w += NTH) dst[w] = __ldcg(src + w);
    if (posed) {
      for (int w = tid; w < nst; w += NTH) {
        const int q = w / A, i = w - q * A;
        stage[w] = __ldcg(base_scr + (size_t)q * DS_MAX_ATOMS + i);
      }
      for (int w = tid; w < nrt; w += NTH) srt[w] = __ldcg(out.rtors + (size_t)f0 * N + w);
    }
  }
  __syncthreads();
  MARK2(1, lig * dp.N + r);
  const LatRec *lr = T.rec;
  // warp 0, lane = restart: the counters in the oracle's sequential order (restarts run in order
  // and a DegenerateAxis stops the ligand, so only restarts up to the first degenerate one count,
  // P14), and the valid restarts in (geom desc, restart asc) order; the others tabulate the pairs
  if (tid < 32) {
    const bool in = tid < N;
    const int val = in ? lr[tid].valid : 0, gq = in ? lr[tid].geom : 0;
    const unsigned dgm = __ballot_sync(kFull, in && lr[tid].degen);
    const int nal = dgm ? __ffs((int)dgm) : N;
    const bool cnt = tid < nal;
    const unsigned ev = __reduce_add_sync(kFull, cnt ? lr[tid].evals : 0u);
    const unsigned pr = __reduce_add_sync(kFull, cnt ? lr[tid].pairs : 0u);
    const unsigned ex = __reduce_add_sync(kFull, cnt ? lr[tid].exits : 0u);
    const unsigned vm = __ballot_sync(kFull, val);
    int rank = 0;
    for (int q = 0; q < N; ++q) {
      const int gp = __shfl_sync(kFull, gq, q);
      rank += ((vm >> q) & 1u) && (gp > gq || (gp == gq && q < tid));
    }
    if (val) T.ord[rank] = tid;
    if (in) T.dis[tid] = 0u;
    if (tid == 0) {
      T.s_cnt[0] = ev;
      T.s_cnt[1] = pr;
      T.s_cnt[2] = ex;
      T.s_cnt[3] = dgm != 0u;
      T.s_nal = (unsigned)nal;
      T.s_degf = dgm ? lr[nal - 1].degen_f : 0;
      T.nvp = __popc(vm);  // the valid restarts
    }
  } else {
    for (int pidx = tid - 32; pidx < npairs; pidx += NTH - 32) {
      int p = 0, rem = pidx;
      while (rem >= N - 1 - p) {
        rem -= N - 1 - p;
        ++p;
      }
      T.vp[pidx] = (uint16_t)(p | (p + 1 + rem) << 8);
    }
  }
  __syncthreads();
  ds_result res;
  memset(&res, 0, sizeof res);
  res.poses_scored = T.s_nal * (unsigned)dp.n_rot + T.s_cnt[0];
  res.bump_checks = T.s_cnt[1];
  res.bump_early_exits = T.s_cnt[2];
  if (T.s_cnt[3]) {
    res.status = DS_STATUS_DEGENERATE_AXIS;
    if (tid == 0) out.res[lig] = res;
    // the sequential oracle stops at restart rd, fragment fd: later records stay zero
    const int rd = (int)T.s_nal - 1, fd = T.s_degf;
    if (out.rrec)
      for (int q = rd + tid; q < N; q += NTH) {
        ds_restart_record z;
        memset(&z, 0, sizeof z);
        out.rrec[(size_t)lig * N + q] = z;
      }
    for (int q = tid; q < nrt; q += NTH) {
      const int f = q / N, rr = q - f * N;
      uint8_t v = __ldcg(out.rtors + (size_t)f0 * N + q);
      if (rr > rd || (rr == rd && f >= fd)) {
        v = 0;
        out.rtors[(size_t)f0 * N + q] = 0;
      }
      if (out.rtors_host) out.rtors_host[(size_t)f0 * N + q] = v;
    }
    return;
  }
  const int nvalid = T.nvp;
  if (nvalid == 0) {
    res.status = DS_STATUS_NO_VALID_POSE;
    if (tid == 0) out.res[lig] = res;
    return;
  }
  const int heavy = T.heavy;
  const double lim = __dmul_rn(dp.thr2, (double)heavy);
  // RMSD of every valid pair (P12), a warp per pair.  The oracle compares its sequential f64 sum
  // over the heavy atoms in atom order with thr2 * heavy; the lanes make the per-atom terms of 32
  // atoms at once (hydrogens contribute +0.0, an exact no-op) and a tree sum T of them.  T and the
  // sequential sum both lie within n u S of the exact sum S of the same terms (n <= 160 terms,
  // u = 2^-53, so within 2e-14 S of each other), so a margin of 1e-12 relative decides the
  // comparison exactly; only a pair inside the margin runs the sequential sum (every lane adds the
  // terms in atom order from shuffles).
  {
    const int lane = tid & 31;
    for (int k = tid >> 5; k < npairs; k += NTH / 32) {
      const int p = T.vp[k] & 0xFF, q = T.vp[k] >> 8;
      if (!lr[p].valid || !lr[q].valid) continue;
      double t[(DS_MAX_ATOMS + 31) / 32];
      double part = 0.0;
#pragma unroll
      for (int c = 0; c < (DS_MAX_ATOMS + 31) / 32; ++c) {
        const int i = 32 * c + lane;
        t[c] = 0.0;
        if (i < A)
          t[c] = posed ? rmsd_term(stage[p * A + i], stage[q * A + i])
                       : rmsd_term(__ldcg(base_scr + (size_t)p * DS_MAX_ATOMS + i),
                                   __ldcg(base_scr + (size_t)q * DS_MAX_ATOMS + i));
        part = __dadd_rn(part, t[c]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(kFull, part, o));
      bool dis;
      if (__dmul_rn(part, 1.0 - 1e-12) >= lim) {
        dis = true;
      } else if (__dmul_rn(part, 1.0 + 1e-12) < lim) {
        dis = false;
      } else {
        double sum = 0.0;
#pragma unroll
        for (int c = 0; c < (DS_MAX_ATOMS + 31) / 32; ++c)
          if (32 * c < A)
#pragma unroll
            for (int j = 0; j < 32; ++j) sum = __dadd_rn(sum, __shfl_sync(kFull, t[c], j));
        dis = sum >= lim;
      }
      if (lane == 0 && heavy > 0 && dis) {
        atomicOr(&T.dis[p], 1u << q);
        atomicOr(&T.dis[q], 1u << p);
      }
    }
  }
  __syncthreads();
  MARK2(3, lig * dp.N + r);
  // warp 0: the greedy keep in rank order (a candidate is kept when it is dissimilar to every pose
  // kept so far), then the best rescored kept pose (ties -> smallest restart)
  if (tid < 32) {
    const int oc = tid < nvalid ? T.ord[tid] : 0;
    const unsigned od = tid < nvalid ? T.dis[oc] : 0u;
    unsigned km = 0u;
    int nk = 0;
    for (int o = 0; o < nvalid && nk < dp.K; ++o) {
      const int c = __shfl_sync(kFull, oc, o);
      const unsigned d = __shfl_sync(kFull, od, o);
      if ((d & km) == km) {
        if (tid == nk) T.kept[nk] = c;
        km |= 1u << c;
        ++nk;
      }
    }
    __syncwarp();
    const int rr = tid < nk ? T.kept[tid] : 0x7FFFFFFF;
    long long ch = tid < nk ? lr[rr].chem : LLONG_MIN;
    long long bc = ch;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bc = max(bc, __shfl_xor_sync(kFull, bc, o));
    const int br = __reduce_min_sync(kFull, (unsigned)(ch == bc ? rr : 0x7FFFFFFF));
    if (tid < nk && out.rrec) out.rrec[(size_t)lig * N + rr].kept = (uint8_t)(tid + 1);
    if (tid == 0) {
      T.nkept = nk;
      T.s_cnt[0] = (unsigned)br;
      T.chem = (unsigned long long)bc;
    }
  }
  __syncthreads();
  MARK2(4, lig * dp.N + r);
  const int nk = T.nkept, best_r = (int)T.s_cnt[0];
  const long long best_chem = (long long)T.chem;
  const int brot = (int)lr[best_r].rot;
  res.status = DS_STATUS_OK;
  res.geom_score = lr[best_r].geom;
  res.chem_fx = best_chem;
  res.best_restart = (uint8_t)best_r;
  res.best_ax = (uint8_t)(brot / dp.n_a);
  res.best_ay = (uint8_t)(brot - (brot / dp.n_a) * dp.n_a);
  res.n_kept = (uint8_t)nk;
  if (tid == 0) out.res[lig] = res;
  if (out.best_coords)
    for (int i = tid; i < A; i += NTH) {
      const float4 x = posed ? stage[best_r * A + i] : __ldcg(base_scr + (size_t)best_r * DS_MAX_ATOMS + i);
      float *o = out.best_coords + 3 * (size_t)(a0 + i);
      o[0] = __fmaf_rn(x.x, pk.spacing, pk.ox);
      o[1] = __fmaf_rn(x.y, pk.spacing, pk.oy);
      o[2] = __fmaf_rn(x.z, pk.spacing, pk.oz);
    }
  if (out.best_tors)
    for (int f = tid; f < F; f += NTH)
      out.best_tors[f0 + f] = posed ? srt[f * N + best_r] : __ldcg(out.rtors + (size_t)(f0 + f) * N + best_r);
  if (out.rtors_host)  // zero-copy outputs: every restart's torsion indices, straight to the host
    for (int q = tid; q < nrt; q += NTH)
      out.rtors_host[(size_t)f0 * N + q] = posed ? srt[q] : __ldcg(out.rtors + (size_t)f0 * N + q);
  MARK(4, lig * dp.N + r);
}

// kNT: the torsion angle count when it is the default 10 (compile-time sweep layout), 0 = runtime
template <bool kSmemGrid, int kNT>
__global__ void __launch_bounds__(kLatThreads, 1)
    k_optimize_latency(PocketView pk, BatchView bt, DockParams dp, int *scores, const unsigned *keys, OptOut out,
                       LatRec *recs, int *done) {
  __shared__ LatSmem S;
  extern __shared__ __align__(16) unsigned char dsm[];  // [trig 360][fragment records][grid]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lig = blockIdx.x / dp.N, r = blockIdx.x - lig * dp.N;
  MARK(0, blockIdx.x);
  const int a0 = bt.atom_off[lig], A = bt.atom_off[lig + 1] - a0;
  const int f0 = bt.frag_off[lig], F = bt.frag_off[lig + 1] - f0;
  const GridGeom g = pk.g;
  // stage the trig table, this ligand's fragment records, the weights, the bin LUT and (if it
  // fits) the pocket grid with bulk async copies (one thread issues, the TMA engine moves them;
  // ~200 KB would otherwise take 50 dependent load/store rounds of the CTA): the trig table
  // lands on bar[0] (needed for the initial pose), the rest on bar[1], awaited only before the
  // fragment loop so the copies overlap the argmax and the initial pose
  __shared__ __align__(8) unsigned long long bar[2];
  float2 *strig = reinterpret_cast<float2 *>(dsm);
  uint4 *sfrag = reinterpret_cast<uint4 *>(dsm + 360 * sizeof(float2));
  int32_t *sw = reinterpret_cast<int32_t *>(dsm + 360 * sizeof(float2) + 2 * (DS_MAX_ATOMS - 2) * sizeof(uint4));
  uint8_t *slut = reinterpret_cast<uint8_t *>(sw) + lat_w_bytes(pk.nb);
  const uint8_t *grid = kSmemGrid ? dsm + lat_base_bytes(pk.nb, pk.lut_cap) : pk.grid;
  const unsigned wbytes = (unsigned)(DS_N_TYPES * DS_N_TYPES * (pk.nb + 1) * 4);
  const int lut_n = pk.lut_cap + 1, lut_bulk = lut_n & ~15;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
    mbar_expect_tx(&bar[0], 360 * sizeof(float2));
    bulk_g2s(strig, pk.trig, 360 * sizeof(float2), &bar[0]);
    mbar_expect_tx(&bar[1], 32u * F + wbytes + lut_bulk + (kSmemGrid ? pk.grid_bytes : 0));
    if (F) bulk_g2s(sfrag, bt.frags + 2 * (size_t)f0, 32u * F, &bar[1]);
    bulk_g2s(sw, pk.wfx, wbytes, &bar[1]);
    if (lut_bulk) bulk_g2s(slut, pk.bin_lut, lut_bulk, &bar[1]);
    if (kSmemGrid) bulk_g2s(const_cast<uint8_t *>(grid), pk.grid, pk.grid_bytes, &bar[1]);
    S.key = 0u;
    S.pairs = 0u;
    S.degen = 0;
    S.t.geom = 0;
    S.t.heavy = 0;
    S.t.chem = 0ull;
  }
  for (int i = lut_bulk + tid; i < lut_n; i += kLatThreads) slut[i] = __ldg(pk.bin_lut + i);  // < 16 B tail
  __syncthreads();
  // everything above only read inputs that were complete before the alignment kernel started; the
  // keys / scores it writes are read below, after the programmatic-dependent-launch wait (a no-op
  // when the kernel was launched without the attribute)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // ---- argmax of the alignment scores (ties -> smallest rotation index); each slot is zeroed by
  // the thread that read it, so the buffer is clean for the next call (no memset per call) ----
  if (keys) {  // the cluster align kernel already reduced this (ligand, restart) to its key
    if (tid == 0) S.key = __ldcg(keys + (size_t)lig * dp.N + r);
  } else {
    int *sc = scores + ((size_t)lig * dp.N + r) * dp.n_rot;
    unsigned best = 0u;
    for (int q = tid; q < dp.n_rot; q += kLatThreads) {
      best = max(best, ((unsigned)(__ldcg(sc + q) + 32768) << 16) | (unsigned)(65535 - q));
      __stcg(sc + q, 0);
    }
    best = __reduce_max_sync(kFull, best);
    if (lane == 0) atomicMax(&S.key, best);
  }
  __syncthreads();
  mbar_wait(&bar[0], 0);
  const unsigned key = S.key;
  // grid score of the current pose carried along the fragment chain (the aligned pose scores the
  // key's score, a committed angle its key's): a fragment's non-moving atoms score total - the
  // angle-0 sum of its moving atoms, so phase (A) reads no grid value and the end no pass
  int total = (int)(key >> 16) - 32768;
  const int rot = 65535 - (int)(key & 0xFFFFu);
  const int ix = rot / dp.n_a, iy = rot - ix * dp.n_a;
  {
    float R0s[9], T[3], Rp[9];
    start_params(bt.idh[lig], dp.seed, r, strig, pk.inv_s, g.nx, g.ny, g.nz, R0s, T);
    align_rx(strig[ix * dp.step_a], R0s, Rp);
    const float2 cy = strig[iy * dp.step_a];
    for (int i = tid; i < A; i += kLatThreads) {
      const float4 d = __ldg(bt.atoms + a0 + i);
      const float3 u = align_u(align_v(Rp, d.x, d.y, d.z), cy.x, cy.y, T);
      S.u[i] = make_float4(u.x, u.y, u.z, d.w);
    }
  }
  __syncthreads();
  unsigned evals = 0, exits = 0;
  int all_bumped = 0;
  const unsigned lt = lanemask_lt();
  const int nslot = (A + 31) >> 5;
  mbar_wait(&bar[1], 0);
  MARK(1, blockIdx.x);
  for (int f = 0; f < F; ++f) {
    const uint4 fa = sfrag[2 * f];
    const uint4 fb = sfrag[2 * f + 1];
    const int ab = (int)(fb.y & 0xFFu), ae = (int)((fb.y >> 8) & 0xFFu);
    // ---- (A) one phase, one barrier: every thread derives the compaction of M / C' from the
    // fragment's mask words (registers only), builds the axis itself (the same bits in every
    // thread, so the degenerate-axis break is uniform), writes its atom's list slot and
    // cylindrical coordinates, and adds the non-moving atoms' grid values into base[f & 1] ----
    const float4 pa = S.u[ab], pb = S.u[ae];
    const float3 a3 = make_float3(pa.x, pa.y, pa.z);
    float kx = 0.f, ky = 0.f, kz = 0.f;
    if (dp.n_t > 1) {
      const float vx = __fsub_rn(pb.x, pa.x), vy = __fsub_rn(pb.y, pa.y), vz = __fsub_rn(pb.z, pa.z);
      const float len = __fsqrt_rn(__fmaf_rn(vz, vz, __fmaf_rn(vy, vy, __fmul_rn(vx, vx))));
      if (!(len >= dp.eps_axis)) {
        if (tid == 0) {
          S.degen = 1;
          S.degen_f = f;
        }
        break;
      }
      kx = __fdiv_rn(vx, len);
      ky = __fdiv_rn(vy, len);
      kz = __fdiv_rn(vz, len);
    }
    int nM = 0, nC = 0, mpre = 0, cpre = 0;
    unsigned my_bm = 0u, my_bc = 0u;
#pragma unroll
    for (int w = 0; w < 5; ++w) {
      if (w < nslot) {
        const unsigned word = w == 0 ? fa.x : w == 1 ? fa.y : w == 2 ? fa.z : w == 3 ? fa.w : fb.x;
        const int lim = A - 32 * w;
        const unsigned vmask = lim >= 32 ? kFull : ((1u << lim) - 1u);
        const unsigned bm = word & vmask;
        unsigned bc = ~word & vmask;
        if ((ab >> 5) == w) bc &= ~(1u << (ab & 31));
        if ((ae >> 5) == w) bc &= ~(1u << (ae & 31));
        if (w < warp) {
          mpre += __popc(bm);
          cpre += __popc(bc);
        } else if (w == warp) {
          mpre += __popc(bm & lt);
          cpre += __popc(bc & lt);
          my_bm = bm;
          my_bc = bc;
        }
        nM += __popc(bm);
        nC += __popc(bc);
      }
    }
    if (tid < A) {
      const float4 p = S.u[tid];
      if ((my_bm >> lane) & 1u) {
        S.mlist[mpre] = (uint8_t)tid;
        S.chm[mpre] = lat_cyl(p, a3, kx, ky, kz);
        S.cn[mpre] = 0;
      } else if ((my_bc >> lane) & 1u) {
        S.clist[cpre] = (uint8_t)tid;
        S.chr[cpre] = lat_cyl(p, a3, kx, ky, kz);
      }
    }
    if (tid < 32) {
      S.ascore[tid] = 0;
      S.bcode[tid] = 0x7FFFFFFF;
    }
    if (tid == 0) S.abump = 0u;
    __syncthreads();
    // ---- (C) bump candidates: every (moving, complement) pair over all threads (cylindrical
    // bound, see ds_optimize.cu) ----
    if (nC > 0) {
      const int total = nM * nC;
      int pm = small_div(tid, nC), pc = tid - pm * nC;
      const int dm = small_div(kLatThreads, nC), dc = kLatThreads - dm * nC;
      for (int p0 = 0; p0 < total; p0 += kLatThreads) {
        if (p0 + tid < total) {
          const float2 hm = S.chm[pm], hc = S.chr[pc];
          const float dh = hm.x - hc.x, dr = hm.y - hc.y;
          if (dh * dh + dr * dr < dp.cull2) {
            const unsigned k = atomicAdd(&S.cn[pm], 1u);
            if (k < (unsigned)kLatCand) S.cl[pm][k] = S.clist[pc];
          }
        }
        pm += dm;
        pc += dc;
        if (pc >= nC) {
          pc -= nC;
          ++pm;
        }
      }
    }
    __syncthreads();
    // ---- (D) the angle sweep: thread = (angle a, moving-atom group mg); rotation and partial score
    // in registers over m = mg, mg + G, ...; one shared atomic per thread at the end ----
    unsigned best_key = 0u;
    int base = 0;  // score of the atoms the torsion does not move
    const int n_t = kNT ? kNT : dp.n_t;
    for (int k0 = 0; k0 < n_t; k0 += 32) {
      const int nA = kNT ? kNT : min(32, n_t - k0);
      if (k0 > 0) {
        __syncthreads();
        if (tid < 32) {
          S.ascore[tid] = 0;
          S.bcode[tid] = 0x7FFFFFFF;
        }
        if (tid == 0) S.abump = 0u;
        __syncthreads();
      }
      // thread = (angle a, group mg), exact reciprocal division (no integer divide on the chain)
      const int G = kNT ? kLatThreads / kNT : small_div(kLatThreads, nA);
      const int mg = kNT ? tid / kNT : small_div(tid, nA), a = tid - mg * nA;
      if (mg < G) {
        float R[9];
        const int kang = k0 + a;
        if (kang > 0) {
          const float2 cs = strig[kang * dp.step_t];
          torsion_matrix(kx, ky, kz, cs.x, cs.y, R);
        }
        int part = 0;
        bool hit_any = false;
        // two moving atoms per step (independent chains: twice the loads in flight); a bump on
        // either marks the angle, whose partial score is then never read
        // early exit: a thread stops once its next atom lies beyond the first bumping slot found so far
        // for its angle; every slot up to the sequential scan's first bump is then tested, so the
        // minimum (and the pair count derived from it) is independent of thread timing (P14)
        // angle 0 always runs to the end: its complete sum gives the non-moving atoms' score
        for (int m = mg; m < nM; m += 2 * G) {
          if (dp.early_exit && kang != 0 && (hit_any || m > *(volatile int *)&S.bcode[a])) break;
          const bool two = m + G < nM;
          const int m1 = two ? m + G : m;
          const float4 p0 = S.u[S.mlist[m]], p1 = S.u[S.mlist[m1]];
          const float3 q0 = kang == 0 ? make_float3(p0.x, p0.y, p0.z) : torsion_apply(R, a3, p0.x, p0.y, p0.z);
          const float3 q1 = kang == 0 ? make_float3(p1.x, p1.y, p1.z) : torsion_apply(R, a3, p1.x, p1.y, p1.z);
          const int gv0 = lat_grid_val<kSmemGrid>(grid, node_index(g, q0.x, q0.y, q0.z));
          const int gv1 = lat_grid_val<kSmemGrid>(grid, node_index(g, q1.x, q1.y, q1.z));
          const float d0 = lat_min_d2(S, m, nC, q0), d1 = lat_min_d2(S, m1, nC, q1);
          const bool hit = d0 < dp.bd2 || d1 < dp.bd2;
          if (hit) {
            hit_any = true;
            atomicOr(&S.abump, 1u << a);
            if (dp.early_exit) atomicMin(&S.bcode[a], d0 < dp.bd2 ? m : m1);
          }
          if (!hit || kang == 0) part += two ? gv0 + gv1 : gv0;
        }
        if (part) atomicAdd(&S.ascore[a], part);
      }
      __syncthreads();
      // pairs evaluated at moving-row granularity (P14): the whole rows of the moving slots up to
      // and including the first bumping one, or all nM * nC
      if (warp == 0) {
        unsigned np = 0;
        if (lane < nA) {
          const int mb = S.bcode[lane];
          np = (dp.early_exit && mb != 0x7FFFFFFF) ? (unsigned)((mb + 1) * nC) : (unsigned)(nM * nC);
        }
        np = __reduce_add_sync(kFull, np);
        if (lane == 0) S.pairs += np;
      }
      // ---- (E) best clean angle, computed by every warp (no extra barrier) ----
      const unsigned abump = S.abump;
      unsigned kk = 0;
      if (k0 == 0) base = total - S.ascore[0];
      if (lane < nA && !((abump >> lane) & 1u))
        kk = ((unsigned)(base + S.ascore[lane] + 32768) << 16) | (unsigned)(65535 - (k0 + lane));
      best_key = max(best_key, __reduce_max_sync(kFull, kk));
      evals += (unsigned)nA;
      if (dp.early_exit) exits += (unsigned)__popc(abump);
    }
    const int best_k = best_key ? 65535 - (int)(best_key & 0xFFFFu) : -1;
    if (best_key) total = (int)(best_key >> 16) - 32768;  // the committed pose's score
    if (tid == 0) out.rtors[(size_t)(f0 + f) * dp.N + r] = best_k < 0 ? (uint8_t)DS_TORSION_NONE : (uint8_t)best_k;
    if (best_k > 0)
      for (int m = tid; m < nM; m += kLatThreads) {
        const int i = S.mlist[m];
        const float4 p = S.u[i];
        const float3 q = lat_torsion_pos(strig, dp.step_t, best_k, kx, ky, kz, a3, p);
        S.u[i] = make_float4(q.x, q.y, q.z, p.w);
      }
    if (best_k < 0) ++all_bumped;
    __syncthreads();
  }
  __syncthreads();  // S.degen (a degenerate axis breaks every thread out at the same fragment)
  MARK(2, blockIdx.x);
  lat_tail<kLatThreads, true>(S.t, S.u, S.degen, S.degen_f, total, !(F >= 1 && all_bumped == F), key, ix, iy, rot, evals,
                        S.pairs, exits, pk, dp, sw, slut, out, recs, done, lig, r, a0, A, f0, F,
                        kSmemGrid ? reinterpret_cast<float4 *>(const_cast<uint8_t *>(grid)) : nullptr,
                        kSmemGrid ? pk.grid_bytes : 0);
}

// ==== cluster-speculative optimisation: one (ligand, restart) over a cluster of n_t CTAs ==========
// The fragment chain is the latency family's critical path (~2.4 us per fragment of dependent,
// barrier-separated phases on one SM).  Fragment f + 1 depends on f only through the angle f
// commits, and there are n_t of those (every angle bumped = no commit = angle 0's positions), so
// a cluster evaluates fragments in pairs.  The lead (thread group 0 of CTA 0) sweeps f on the
// current pose; thread group 1 of CTA h commits angle h of f on a copy of the pose and sweeps
// f + 1 on it, concurrently.  The lead publishes its outcome for f into every CTA's shared memory
// (DSMEM stores, each followed by a release arrive on that CTA's mbarrier); group 1 of CTA a_f
// (CTA 0 when every angle of f bumped), the winner, then pushes its pose — f and f + 1 committed
// — and its outcome for f + 1 the same way, and every CTA moves on to f + 2 as soon as that one
// push has landed: the losing hypotheses are never waited for.  Half the chain length, on
// n_t x N SMs instead of N; bit-identical to the sequential chain (the pose is the winner's,
// computed by the same operations).  Ordering: the pose is double-buffered, and the lead
// publishes a_f only after every hypothesis group has signalled (rbar) that it has read the
// step's pose, so a push never overwrites a buffer that is still being read.  (Group 0 of
// CTAs 1 .. n_t - 1 idles: 1 + n_t single-group CTAs would not all be resident — one GPC of the
// B200 holds fewer than 11 CTAs of this size, so only 7 such clusters fit.)
constexpr int kSpecH = 10;             // hypotheses per fragment = torsion angles = cluster size
constexpr int kSpecT = 256;            // threads per group (two groups per CTA)
constexpr int kAlignR = 900 / kSpecH;  // alignment rotations per CTA (n_a = 30): 3 ax x 30 ay
constexpr int kAlignG = 11;            // atom groups per (ax, ay pair) (3 x 15 x kAlignG <= 2 kSpecT)

struct LatGrp {                        // a CTA's per-fragment scratch
  float2 chr[DS_MAX_ATOMS];
  float2 chm[DS_MAX_ATOMS];
  uint8_t mlist[DS_MAX_ATOMS];
  uint8_t clist[DS_MAX_ATOMS];
  uint8_t cl[DS_MAX_ATOMS][kLatCand];
  unsigned cn[DS_MAX_ATOMS];
  int ascore[32];
  int bcode[32];
  unsigned abump;
};

// one fragment's outcome packed into 64 bits, so that a single (single-copy atomic) DSMEM store
// carries it together with its validity tag:
//   [0, 8) tag = step + 1   [8] degenerate axis   [9, 13) committed angle + 1 (0: every angle bumped)
//   [13, 18) early exits    [18, 36) score change of the committed angle + 2^17   [36, 64) P14 pairs
struct SpecRec {
  int best_k, delta, degen;
  unsigned pairs, exits;
};
__device__ __forceinline__ unsigned long long spec_pack(unsigned tag, int degen, int best_k, int delta, unsigned pairs,
                                                        unsigned exits) {
  return (unsigned long long)tag | (unsigned long long)degen << 8 | (unsigned long long)(best_k + 1) << 9 |
         (unsigned long long)exits << 13 | (unsigned long long)(delta + 131072) << 18 | (unsigned long long)pairs << 36;
}
__device__ __forceinline__ SpecRec spec_unpack(unsigned long long v) {
  SpecRec r;
  r.degen = (int)((v >> 8) & 1u);
  r.best_k = (int)((v >> 9) & 15u) - 1;
  r.exits = (unsigned)((v >> 13) & 31u);
  r.delta = (int)((v >> 18) & 0x3FFFFu) - 131072;
  r.pairs = (unsigned)(v >> 36);
  return r;
}

__device__ __forceinline__ void grp_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(kSpecT) : "memory");
}
// the shared::cluster address of p in CTA rank
__device__ __forceinline__ unsigned dsmem(const void *p, unsigned rank) {
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_addr(p)), "r"(rank));
  return ra;
}
// publish a tagged 64-bit record into CTA rank's slot, and wait for this CTA's slot to carry tag.
// A slot is zeroed at kernel start (before a cluster barrier) and written once; the record
// travels in the same single-copy-atomic word as its validity tag, so relaxed cluster-scope
// (strong) accesses suffice and no fence is needed.  compute-sanitizer racecheck reports these
// pairs (it orders cross-CTA shared-memory accesses by cluster barriers only); DESIGN.md §8.
__device__ __forceinline__ void slot_put(unsigned long long *slot, unsigned rank, unsigned long long v) {
  asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(dsmem(slot, rank)), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long slot_get(unsigned long long *slot, unsigned tag) {
  unsigned long long v;
  do {
    asm volatile("ld.relaxed.cluster.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(smem_addr(slot)) : "memory");
  } while ((unsigned)(v & 0xFFu) != tag);
  return v;
}
__device__ __forceinline__ void mbar_wait_cluster(unsigned long long *bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAITC:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONEC;\n\tbra LAB_WAITC;\n\tDONEC:\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// the torsion axis of a fragment from the positions U (the recipe of the sequential kernel);
// false when it is degenerate
__device__ __forceinline__ bool lat_axis(const float4 *U, int ab, int ae, float eps, float3 &a3, float &kx, float &ky,
                                         float &kz) {
  const float4 pa = U[ab], pb = U[ae];
  a3 = make_float3(pa.x, pa.y, pa.z);
  const float vx = __fsub_rn(pb.x, pa.x), vy = __fsub_rn(pb.y, pa.y), vz = __fsub_rn(pb.z, pa.z);
  const float len = __fsqrt_rn(__fmaf_rn(vz, vz, __fmaf_rn(vy, vy, __fmul_rn(vx, vx))));
  if (!(len >= eps)) return false;
  kx = __fdiv_rn(vx, len);
  ky = __fdiv_rn(vy, len);
  kz = __fdiv_rn(vz, len);
  return true;
}

__device__ __forceinline__ unsigned frag_word(uint4 fa, uint4 fb, int w) {
  return w == 0 ? fa.x : w == 1 ? fa.y : w == 2 ? fa.z : w == 3 ? fa.w : fb.x;
}

// nearest bump candidate of moving atom m at q (lat_min_d2 over a group's scratch)
__device__ __forceinline__ float grp_min_d2(const float4 *U, const LatGrp &S, int m, int nC, float3 q) {
  float mind = __int_as_float(0x7f800000);
  const unsigned cnt = S.cn[m];
  if (cnt <= (unsigned)kLatCand) {
    for (unsigned t = 0; t < cnt; ++t) {
      const float4 y = U[S.cl[m][t]];
      mind = fminf(mind, dist2(q.x, q.y, q.z, y.x, y.y, y.z));
    }
  } else {
    for (int c = 0; c < nC; ++c) {
      const float4 y = U[S.clist[c]];
      mind = fminf(mind, dist2(q.x, q.y, q.z, y.x, y.y, y.z));
    }
  }
  return mind;
}

// one fragment's phases (A) compaction + cylindrical coordinates, (C) bump candidates, (D) the
// angle sweep, (E) best clean angle, by the kSpecT threads of a CTA (gt = thread index,
// barrier id bar) on the positions U, which it does not modify.  Returns the committed angle
// (-1: all bumped, -2: degenerate axis), the same in every thread of the group; the group's
// lanes of warp 0 get the packed outcome (spec_pack; the tag is the caller's).  The axis and the
// moving count are left for the caller's commit.
template <bool kSmemGrid>
__device__ __forceinline__ int lat_frag(const float4 *U, LatGrp &S, uint4 fa, uint4 fb, int A, const GridGeom &g,
                                        const uint8_t *grid, const float2 *strig, const DockParams &dp, int gt,
                                        int bar, unsigned long long &rec, float3 &a3, float &kx, float &ky, float &kz,
                                        int &nMo) {
  constexpr int kNT = kSpecH;
  const int lane = gt & 31, warp = gt >> 5;
  const int ab = (int)(fb.y & 0xFFu), ae = (int)((fb.y >> 8) & 0xFFu);
  if (!lat_axis(U, ab, ae, dp.eps_axis, a3, kx, ky, kz)) {
    rec = spec_pack(0, 1, -1, 0, 0u, 0u);
    return -2;
  }
  // ---- (A) ----
  const unsigned lt = lanemask_lt();
  const int nslot = (A + 31) >> 5;
  int nM = 0, nC = 0, mpre = 0, cpre = 0;
  unsigned my_bm = 0u, my_bc = 0u;
#pragma unroll
  for (int w = 0; w < 5; ++w) {
    if (w < nslot) {
      const unsigned word = frag_word(fa, fb, w);
      const int lim = A - 32 * w;
      const unsigned vmask = lim >= 32 ? kFull : ((1u << lim) - 1u);
      const unsigned bm = word & vmask;
      unsigned bc = ~word & vmask;
      if ((ab >> 5) == w) bc &= ~(1u << (ab & 31));
      if ((ae >> 5) == w) bc &= ~(1u << (ae & 31));
      if (w < warp) {
        mpre += __popc(bm);
        cpre += __popc(bc);
      } else if (w == warp) {
        mpre += __popc(bm & lt);
        cpre += __popc(bc & lt);
        my_bm = bm;
        my_bc = bc;
      }
      nM += __popc(bm);
      nC += __popc(bc);
    }
  }
  if (gt < A) {
    const float4 p = U[gt];
    if ((my_bm >> lane) & 1u) {
      S.mlist[mpre] = (uint8_t)gt;
      S.chm[mpre] = lat_cyl(p, a3, kx, ky, kz);
      S.cn[mpre] = 0;
    } else if ((my_bc >> lane) & 1u) {
      S.clist[cpre] = (uint8_t)gt;
      S.chr[cpre] = lat_cyl(p, a3, kx, ky, kz);
    }
  }
  if (gt < 32) {
    S.ascore[gt] = 0;
    S.bcode[gt] = 0x7FFFFFFF;
  }
  if (gt == 0) S.abump = 0u;
  grp_sync(bar);
  // ---- (C) ----
  if (nC > 0) {
    const int total = nM * nC;
    int pm = small_div(gt, nC), pc = gt - pm * nC;
    const int dm = small_div(kSpecT, nC), dc = kSpecT - dm * nC;
    for (int p0 = 0; p0 < total; p0 += kSpecT) {
      if (p0 + gt < total) {
        const float2 hm = S.chm[pm], hc = S.chr[pc];
        const float dh = hm.x - hc.x, dr = hm.y - hc.y;
        if (dh * dh + dr * dr < dp.cull2) {
          const unsigned k = atomicAdd(&S.cn[pm], 1u);
          if (k < (unsigned)kLatCand) S.cl[pm][k] = S.clist[pc];
        }
      }
      pm += dm;
      pc += dc;
      if (pc >= nC) {
        pc -= nC;
        ++pm;
      }
    }
  }
  grp_sync(bar);
  // ---- (D) thread = (angle a, moving-atom group mg), as in k_optimize_latency ----
  {
    constexpr int G = kSpecT / kNT;
    const int mg = gt / kNT, a = gt - mg * kNT;
    if (mg < G) {
      float R[9];
      if (a > 0) {
        const float2 cs = strig[a * dp.step_t];
        torsion_matrix(kx, ky, kz, cs.x, cs.y, R);
      }
      int part = 0;
      bool hit_any = false;
      for (int m = mg; m < nM; m += 2 * G) {
        if (dp.early_exit && a != 0 && (hit_any || m > *(volatile int *)&S.bcode[a])) break;
        const bool two = m + G < nM;
        const int m1 = two ? m + G : m;
        const float4 p0 = U[S.mlist[m]], p1 = U[S.mlist[m1]];
        const float3 q0 = a == 0 ? make_float3(p0.x, p0.y, p0.z) : torsion_apply(R, a3, p0.x, p0.y, p0.z);
        const float3 q1 = a == 0 ? make_float3(p1.x, p1.y, p1.z) : torsion_apply(R, a3, p1.x, p1.y, p1.z);
        const int gv0 = lat_grid_val<kSmemGrid>(grid, node_index(g, q0.x, q0.y, q0.z));
        const int gv1 = lat_grid_val<kSmemGrid>(grid, node_index(g, q1.x, q1.y, q1.z));
        const float d0 = grp_min_d2(U, S, m, nC, q0), d1 = grp_min_d2(U, S, m1, nC, q1);
        const bool hit = d0 < dp.bd2 || d1 < dp.bd2;
        if (hit) {
          hit_any = true;
          atomicOr(&S.abump, 1u << a);
          if (dp.early_exit) atomicMin(&S.bcode[a], d0 < dp.bd2 ? m : m1);
        }
        if (!hit || a == 0) part += two ? gv0 + gv1 : gv0;
      }
      if (part) atomicAdd(&S.ascore[a], part);
    }
  }
  grp_sync(bar);
  // ---- (E) best clean angle by the score change against angle 0 (the non-moving atoms' score is
  // common to every angle), every warp redundantly; P14 pair rows by warp 0 ----
  const unsigned abump = S.abump;
  unsigned kk = 0u;
  if (lane < kNT && !((abump >> lane) & 1u))
    kk = ((unsigned)(S.ascore[lane] - S.ascore[0] + 65536) << 8) | (unsigned)(255 - lane);
  const unsigned best = __reduce_max_sync(kFull, kk);
  const int best_k = best ? 255 - (int)(best & 0xFFu) : -1;
  if (warp == 0) {
    unsigned np = 0;
    if (lane < kNT) {
      const int mb = S.bcode[lane];
      np = (dp.early_exit && mb != 0x7FFFFFFF) ? (unsigned)((mb + 1) * nC) : (unsigned)(nM * nC);
    }
    np = __reduce_add_sync(kFull, np);
    rec = spec_pack(0, 0, best_k, best ? (int)(best >> 8) - 65536 : 0, np, dp.early_exit ? (unsigned)__popc(abump) : 0u);
  }
  nMo = nM;
  return best_k;
}

// commit angle k (> 0) of the fragment whose moving atoms are S.mlist[0 .. nM) into U
__device__ __forceinline__ void lat_commit(float4 *U, const LatGrp &S, int nM, const float2 *strig, int step_t, int k,
                                           float3 a3, float kx, float ky, float kz, int t0, int nth) {
  for (int m = t0; m < nM; m += nth) {
    const int i = S.mlist[m];
    const float4 p = U[i];
    const float3 q = lat_torsion_pos(strig, step_t, k, kx, ky, kz, a3, p);
    U[i] = make_float4(q.x, q.y, q.z, p.w);
  }
}

template <bool kSmemGrid>
__global__ void __launch_bounds__(2 * kSpecT, 1)
    k_optimize_latency_spec(PocketView pk, BatchView bt, DockParams dp, OptOut out, LatRec *recs, int *done) {
  constexpr int NTH = 2 * kSpecT;
  constexpr int kSteps = (DS_MAX_ATOMS - 2 + 1) / 2;
  __shared__ __align__(16) float4 P[DS_MAX_ATOMS];  // the committed pose (every CTA its own copy)
  __shared__ __align__(16) float4 Q[DS_MAX_ATOMS];  // the hypothesis group's pose
  __shared__ LatGrp GS[2];                          // [0]: the lead (CTA 0), [1]: the hypothesis group
  // published outcomes, one slot per step (written once, so never overwritten while unread):
  // slot0: the lead's for f, slot1: the winner's for f + 1
  __shared__ unsigned long long slot0[kSteps], slot1[kSteps];
  __shared__ unsigned long long kslot[kSpecH];      // every CTA's best alignment key
  __shared__ int apart[kAlignG][kAlignR];           // alignment partial scores (atom group, rotation)
  __shared__ LatTail T;
  __shared__ unsigned s_key;
  __shared__ __align__(8) unsigned long long bar[2];
  extern __shared__ __align__(16) unsigned char dsm[];
  cg::cluster_group cl = cg::this_cluster();
  const int h = (int)cl.block_rank();
  const int tid = threadIdx.x, grp = tid / kSpecT, gt = tid - grp * kSpecT;
  const bool lead = h == 0 && grp == 0, hyp = grp == 1;
  const int lr = blockIdx.x / kSpecH;
  const int lig = lr / dp.N, r = lr - lig * dp.N;
  if (h == 0) MARK(0, lr);
  const int a0 = bt.atom_off[lig], A = bt.atom_off[lig + 1] - a0;
  const int f0 = bt.frag_off[lig], F = bt.frag_off[lig + 1] - f0;
  const GridGeom g = pk.g;
  float2 *strig = reinterpret_cast<float2 *>(dsm);
  uint4 *sfrag = reinterpret_cast<uint4 *>(dsm + 360 * sizeof(float2));
  int32_t *sw = reinterpret_cast<int32_t *>(dsm + 360 * sizeof(float2) + 2 * (DS_MAX_ATOMS - 2) * sizeof(uint4));
  uint8_t *slut = reinterpret_cast<uint8_t *>(sw) + lat_w_bytes(pk.nb);
  const uint8_t *grid = kSmemGrid ? dsm + lat_base_bytes(pk.nb, pk.lut_cap) : pk.grid;
  const unsigned wbytes = (unsigned)(DS_N_TYPES * DS_N_TYPES * (pk.nb + 1) * 4);
  const int lut_n = pk.lut_cap + 1, lut_bulk = lut_n & ~15;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
    mbar_expect_tx(&bar[0], 360 * sizeof(float2));
    bulk_g2s(strig, pk.trig, 360 * sizeof(float2), &bar[0]);
    mbar_expect_tx(&bar[1], 32u * F + wbytes + lut_bulk + pk.grid_bytes);
    if (F) bulk_g2s(sfrag, bt.frags + 2 * (size_t)f0, 32u * F, &bar[1]);
    bulk_g2s(sw, pk.wfx, wbytes, &bar[1]);
    if (lut_bulk) bulk_g2s(slut, pk.bin_lut, lut_bulk, &bar[1]);
    T.geom = 0;
    T.heavy = 0;
    T.chem = 0ull;
  }
  for (int i = tid; i < kSteps; i += NTH) {
    slot0[i] = 0ull;
    slot1[i] = 0ull;
  }
  if (tid < kSpecH) kslot[tid] = 0ull;
  if (tid == 0) s_key = 0u;
  for (int i = lut_bulk + tid; i < lut_n; i += NTH) slut[i] = __ldg(pk.bin_lut + i);
  cl.sync();  // every CTA's barriers are initialised and slots cleared before any remote write
  if (h == 0) MARK2(5, lr);
  // the pocket grid: CTA h fetches slice h once and the TMA engine multicasts it into all the
  // cluster's CTAs (each CTA's bar[1] counts the whole grid): 1/10 of the L2 reads
  if (tid == 0) {
    const unsigned sl = ((unsigned)pk.grid_bytes / kSpecH + 15u) & ~15u;
    const unsigned lo = min((unsigned)pk.grid_bytes, h * sl), hi = min((unsigned)pk.grid_bytes, lo + sl);
    if (hi > lo)
      bulk_g2s_multicast(const_cast<uint8_t *>(grid) + lo, pk.grid + lo, hi - lo, &bar[1], (1u << kSpecH) - 1u);
  }
  if (tid < A) Q[tid] = __ldg(bt.atoms + a0 + tid);  // the ligand's atoms (for the alignment)
  mbar_wait(&bar[0], 0);
  // ---- alignment (Alg. 1 lines 4-7, P6) spread over the cluster: CTA h scores the 90 rotations
  // of ax in [3 h, 3 h + 3); a thread takes one ax, a pair of ay (v = R' d shared, the two angles'
  // x / z coordinates in packed f32x2 arithmetic, each lane bit-identical to the scalar recipe)
  // and every kAlignG-th atom; integer sums, so the split does not change them.  Every CTA
  // publishes its best key into every CTA and all take the maximum: the cluster alignment
  // kernel's key. ----
  float R0s[9], Tt[3];
  start_params(bt.idh[lig], dp.seed, r, strig, pk.inv_s, g.nx, g.ny, g.nz, R0s, Tt);
  mbar_wait(&bar[1], 0);
  cta_sync_unaligned();  // the atoms in Q
  if (h == 0) MARK2(6, lr);
  if (tid < kAlignG * (kAlignR / 2)) {
    const int j = tid / (kAlignR / 2), pr = tid - j * (kAlignR / 2);  // pr = ax_local * 15 + ay pair
    const int axl = pr / 15, ay = 2 * (pr - axl * 15);
    float Rp[9];
    align_rx(strig[(3 * h + axl) * dp.step_a], R0s, Rp);
    const float2 c0 = strig[ay * dp.step_a], c1 = strig[(ay + 1) * dp.step_a];
    const f2_t C = f2_pack(c0.x, c1.x), S = f2_pack(c0.y, c1.y), NS = f2_pack(-c0.y, -c1.y);
    const f2_t TX = f2_pack(Tt[0], Tt[0]), TZ = f2_pack(Tt[2], Tt[2]), MM = f2_pack(kMagic, kMagic);
    const unsigned K = (unsigned)(kMagicBits - 1);
    int s0 = 0, s1 = 0;
#pragma unroll 4
    for (int i = j; i < A; i += kAlignG) {
      const float4 d = Q[i];
      const float3 v = align_v(Rp, d.x, d.y, d.z);
      const unsigned yk = g.NX * clamp_bits(__fadd_rn(v.y, Tt[1]), g.by);
      const f2_t VX = f2_pack(v.x, v.x), VZ = f2_pack(v.z, v.z);
      float mx0, mx1, mz0, mz1;
      f2_unpack(f2_add(f2_fma(S, VZ, f2_fma(C, VX, TX)), MM), mx0, mx1);
      f2_unpack(f2_add(f2_fma(C, VZ, f2_fma(NS, VX, TZ)), MM), mz0, mz1);
      const unsigned i0 = min((unsigned)__float_as_int(mx0) - K, g.bx) + g.NXY * min((unsigned)__float_as_int(mz0) - K, g.bz) + yk;
      const unsigned i1 = min((unsigned)__float_as_int(mx1) - K, g.bx) + g.NXY * min((unsigned)__float_as_int(mz1) - K, g.bz) + yk;
      s0 += lat_grid_val<true>(grid, (int)i0);
      s1 += lat_grid_val<true>(grid, (int)i1);
    }
    apart[j][axl * 30 + ay] = s0;
    apart[j][axl * 30 + ay + 1] = s1;
  }
  __syncthreads();
  if (tid < 32 * ((kAlignR + 31) / 32)) {
    unsigned best = 0u;
    if (tid < kAlignR) {
      int sc = 0;
#pragma unroll
      for (int j = 0; j < kAlignG; ++j) sc += apart[j][tid];
      best = ((unsigned)(sc + 32768) << 16) | (unsigned)(65535 - (h * kAlignR + tid));
    }
    best = __reduce_max_sync(kFull, best);
    if ((tid & 31) == 0) atomicMax(&s_key, best);
  }
  __syncthreads();
  if (h == 0) MARK2(7, lr);
  if (tid < kSpecH) slot_put(&kslot[h], tid, (unsigned long long)s_key << 32 | 0xA5u);
  unsigned key = 0u;
  for (int c = 0; c < kSpecH; ++c) key = max(key, (unsigned)(slot_get(&kslot[c], 0xA5u) >> 32));
  int total = (int)(key >> 16) - 32768;
  const int rot = 65535 - (int)(key & 0xFFFFu);
  const int ix = rot / dp.n_a, iy = rot - ix * dp.n_a;
  if (tid < A) {
    float Rp[9];
    align_rx(strig[ix * dp.step_a], R0s, Rp);
    const float2 cy = strig[iy * dp.step_a];
    const float4 d = Q[tid];
    const float3 u = align_u(align_v(Rp, d.x, d.y, d.z), cy.x, cy.y, Tt);
    P[tid] = make_float4(u.x, u.y, u.z, d.w);
  }
  __syncthreads();
  if (h == 0) MARK(1, lr);
  unsigned evals = 0, exits = 0, pairs = 0;
  int all_bumped = 0, degen = 0, degen_f = 0;
#ifdef DS_SPEC_PROBE
  long long t_step = clock64();
#endif
  for (int f = 0, st = 0; (lead || hyp) && f < F; f += 2, ++st) {
    const unsigned tag = (unsigned)st + 1u;
    const bool two = f + 1 < F;  // uniform over the cluster
    const uint4 fa = sfrag[2 * f], fb = sfrag[2 * f + 1];
    float3 fa3;                   // fragment f's axis (hypothesis group)
    float fkx = 0.f, fky = 0.f, fkz = 0.f;
    if (lead) {
      float3 a3;
      float kx, ky, kz;
      int nM = 0;
      unsigned long long rec = 0ull;
      lat_frag<kSmemGrid>(P, GS[0], fa, fb, A, g, grid, strig, dp, gt, 1, rec, a3, kx, ky, kz, nM);
      if (gt < kSpecH) slot_put(&slot0[st], gt, rec | tag);  // lane c publishes into CTA c
      if (gt == 0) SPROBE(0);
    } else {
      // commit hypothesis h of fragment f on a copy of the pose, then sweep f + 1 on it
      const int ab = (int)(fb.y & 0xFFu), ae = (int)((fb.y >> 8) & 0xFFu);
      const bool ok = lat_axis(P, ab, ae, dp.eps_axis, fa3, fkx, fky, fkz);  // else the lead reports the break
      if (!two) grp_sync(2);  // every thread has read the axis atoms before the commit below
      if (two && ok) {
        if (gt < A) {
          const float4 p = P[gt];
          const bool mv = (frag_word(fa, fb, gt >> 5) >> (gt & 31)) & 1u;
          if (mv && h > 0) {
            const float3 q = lat_torsion_pos(strig, dp.step_t, h, fkx, fky, fkz, fa3, p);
            Q[gt] = make_float4(q.x, q.y, q.z, p.w);
          } else {
            Q[gt] = p;
          }
        }
        grp_sync(2);
        if (gt == 0) SPROBE(1);
        float3 a3;
        float kx, ky, kz;
        int nM = 0;
        unsigned long long rec = 0ull;
        lat_frag<kSmemGrid>(Q, GS[1], sfrag[2 * f + 2], sfrag[2 * f + 3], A, g, grid, strig, dp, gt, 2, rec, a3, kx, ky,
                            kz, nM);
        if (gt == 0) SPROBE(2);
        // the winner (CTA 0 when every angle of f bumped) publishes its outcome for f + 1
        const SpecRec r0 = spec_unpack(slot_get(&slot0[st], tag));
        if (gt == 0) SPROBE(3);
        if (!r0.degen && h == (r0.best_k < 0 ? 0 : r0.best_k) && gt < kSpecH) slot_put(&slot1[st], gt, rec | tag);
      }
    }
    const SpecRec r0 = spec_unpack(slot_get(&slot0[st], tag));
    if (r0.degen) {  // a degenerate axis at f: the chain stops (every group alike)
      degen = 1;
      degen_f = f;
      break;
    }
    SpecRec r1;
    if (two) {
      r1 = spec_unpack(slot_get(&slot1[st], tag));
      if (gt == 0) SPROBE(4);
    }
    // every CTA commits a_f and a_{f+1} on its own pose, with the operations the lead and the
    // winner used (so the bits are theirs); in CTA 0 the hypothesis group does it for both groups
    if (hyp) {
      if (r0.best_k > 0 && gt < A && ((frag_word(fa, fb, gt >> 5) >> (gt & 31)) & 1u)) {
        const float4 p = P[gt];
        const float3 q = lat_torsion_pos(strig, dp.step_t, r0.best_k, fkx, fky, fkz, fa3, p);
        P[gt] = make_float4(q.x, q.y, q.z, p.w);
      }
      if (two && !r1.degen && r1.best_k > 0) {
        grp_sync(2);
        const uint4 ga = sfrag[2 * f + 2], gb = sfrag[2 * f + 3];
        float3 b3;
        float bkx, bky, bkz;
        lat_axis(P, (int)(gb.y & 0xFFu), (int)((gb.y >> 8) & 0xFFu), dp.eps_axis, b3, bkx, bky, bkz);
        grp_sync(2);  // every thread has read the axis atoms before they may move
        if (gt < A && ((frag_word(ga, gb, gt >> 5) >> (gt & 31)) & 1u)) {
          const float4 p = P[gt];
          const float3 q = lat_torsion_pos(strig, dp.step_t, r1.best_k, bkx, bky, bkz, b3, p);
          P[gt] = make_float4(q.x, q.y, q.z, p.w);
        }
      }
    }
    if (h == 0)
      __syncthreads();  // CTA 0: the lead reads the committed pose next
    else
      grp_sync(2);
    if (gt == 0) SPROBE(5);
#ifdef DS_SPEC_PROBE
    t_step = clock64();
#endif
    evals += kSpecH;
    pairs += r0.pairs;
    exits += r0.exits;
    all_bumped += r0.best_k < 0;
    if (r0.best_k >= 0) total += r0.delta;
    if (lead && gt == 0)
      out.rtors[(size_t)(f0 + f) * dp.N + r] = r0.best_k < 0 ? (uint8_t)DS_TORSION_NONE : (uint8_t)r0.best_k;
    if (two) {
      if (r1.degen) {
        degen = 1;
        degen_f = f + 1;
        break;
      }
      evals += kSpecH;
      pairs += r1.pairs;
      exits += r1.exits;
      all_bumped += r1.best_k < 0;
      if (r1.best_k >= 0) total += r1.delta;
      if (lead && gt == 0)
        out.rtors[(size_t)(f0 + f + 1) * dp.N + r] = r1.best_k < 0 ? (uint8_t)DS_TORSION_NONE : (uint8_t)r1.best_k;
    }
  }
  // every hypothesis group holds the final pose: the rescore (P11) is split over them and summed
  // into CTA 0 (exact 64-bit integer sum, so the split does not change it)
  const int valid = !(F >= 1 && all_bumped == F);
  if (hyp && !degen && valid) {
    long long acc = lat_rescore_acc(P, A, pk, sw, slut, h * kSpecT + gt, kSpecH * kSpecT);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if ((tid & 31) == 0 && acc) atomicAdd(cl.map_shared_rank(&T.chem, 0), (unsigned long long)acc);
  }
  cl.sync();  // no CTA leaves while another may still access its shared memory
  if (h != 0) return;
  MARK(2, lr);
  lat_tail<NTH, false>(T, P, degen, degen_f, total, valid, key, ix, iy, rot, evals, pairs, exits, pk, dp, sw, slut,
                       out, recs, done, lig, r, a0, A, f0, F,
                       reinterpret_cast<float4 *>(const_cast<uint8_t *>(grid)), pk.grid_bytes);
}

size_t latency_rec_bytes() { return sizeof(LatRec); }

// DS_LATENCY_SPEC: 0 = never the cluster-speculative kernel, 1 = whenever it applies, unset = when
// every (ligand, restart) cluster is resident at once (one ligand spread over the GPU)
static int spec_mode() {
  const char *e = getenv("DS_LATENCY_SPEC");
  return e ? atoi(e) : -1;
}

static int smem_optin() {
  static const int v = [] {
    int dev = 0, x = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&x, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return x;
  }();
  return v;
}

// The cluster-speculative kernel with its own alignment (one launch per call) when it applies:
// the default 12-degree alignment step and 10 torsion angles, the grid in shared memory, and (unless
// forced) every cluster of the call resident at once.  Returns false when the caller must run the
// alignment kernel and the one-CTA chain instead.
bool launch_spread_latency(const PocketView &pk, const BatchView &bt, const DockParams &dp, OptOut out, void *recs,
                           int *done, cudaStream_t st) {
  const int mode = spec_mode();
  if (mode == 0 || dp.n_t != kSpecH || dp.n_a != 30 || dp.step_a <= 0) return false;
  auto kern = k_optimize_latency_spec<true>;
  static const size_t spec_static = [] {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, (const void *)k_optimize_latency_spec<true>);
    cudaFuncSetAttribute((const void *)k_optimize_latency_spec<true>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                         1);
    return (size_t)fa.sharedSizeBytes;
  }();
  const size_t with_grid = lat_base_bytes(pk.nb, pk.lut_cap) + (size_t)pk.grid_bytes;
  if (with_grid + spec_static + 1024 > (size_t)smem_optin()) return false;
  allow_max_smem((const void *)kern);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(bt.L * dp.N * kSpecH);
  cfg.blockDim = dim3(2 * kSpecT);
  cfg.dynamicSmemBytes = with_grid;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kSpecH;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (mode != 1) {  // resident clusters at this shared-memory size (cached per size)
    static std::mutex mu;
    static std::map<size_t, int> resident;
    std::lock_guard<std::mutex> lk(mu);
    auto it = resident.find(with_grid);
    if (it == resident.end()) {
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, (const void *)kern, &cfg) != cudaSuccess) n = 0;
      it = resident.emplace(with_grid, n).first;
    }
    if (bt.L * dp.N > it->second) return false;
  }
  cudaLaunchKernelEx(&cfg, kern, pk, bt, dp, out, (LatRec *)recs, done);
  return true;
}

void launch_optimize_latency(const PocketView &pk, const BatchView &bt, const DockParams &dp, int *scores,
                             const unsigned *keys, OptOut out, void *recs, int *done, bool pdl, cudaStream_t st) {
  const size_t base = lat_base_bytes(pk.nb, pk.lut_cap);
  const size_t with_grid = base + (size_t)pk.grid_bytes;
  const bool fits = with_grid + sizeof(LatSmem) + 1024 <= (size_t)smem_optin();
  const bool nt10 = dp.n_t == 10;
  auto kern = fits ? (nt10 ? k_optimize_latency<true, 10> : k_optimize_latency<true, 0>)
                   : (nt10 ? k_optimize_latency<false, 10> : k_optimize_latency<false, 0>);
  const size_t smem = fits ? with_grid : base;
  allow_max_smem((const void *)kern);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(bt.L * dp.N);
  cfg.blockDim = dim3(kLatThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, pk, bt, dp, scores, keys, out, (LatRec *)recs, done);
}

}  // namespace ds

#ifdef DS_SPEC_PROBE
extern "C" int ds_probe_marks(unsigned long long *out) {
  return (int)cudaMemcpyFromSymbol(out, ds::g_marks, sizeof(ds::g_marks));
}
extern "C" int ds_probe_marks2(unsigned long long *out) {
  return (int)cudaMemcpyFromSymbol(out, ds::g_marks2, sizeof(ds::g_marks2));
}
extern "C" int ds_probe_steps(long long *out) {
  return (int)cudaMemcpyFromSymbol(out, ds::g_steps, sizeof(ds::g_steps));
}
#endif
