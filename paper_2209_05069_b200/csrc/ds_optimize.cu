// Pose optimisation, pose selection and rescoring (Alg. 1 lines 10-21, PAPER.md:227-247;
// SPEC.md:257-285) — batched family, one warp per ligand, as two kernels so
// each gets the whole register file for its own loop nest:
//
// k_torsion_batched — per restart the warp rebuilds the aligned pose from the packed argmax key of
// the alignment kernel, then walks the fragments in list order (they are stateful,
// PAPER.md:278-279).  Per fragment:
//  * ballots compact the moving set M (positions into a per-fragment record array) and the
//    bump-relevant complement C' (not M, not an axis atom);
//  * bump candidates: a torsion keeps each moving atom on its circle about the axis, so (i, j)
//    can only bump if the distance between i's circle and j — sqrt(dh^2 + dr^2) in cylindrical
//    coordinates about the axis — is below the bump distance.  Pairs failing that bound (with a
//    0.02-node margin that dwarfs f32 rounding) are resolved once per fragment instead of once per
//    angle; the survivors (~1.5 % of pairs on the config-3 mix) are recorded with the moving atom
//    (three inline, the rest in a short per-fragment list) and checked exactly with P9 per angle;
//  * all torsion angles at once: lanes own (angle, two moving atoms) slots from a host-built lane
//    table, rotate their atoms with packed f32x2 arithmetic in registers and test their candidates;
//    a hit marks the angle bumped, clean slots add their grid values to base + sum over M
//    (non-moving atoms do not change);
//  * the best clean angle (ties -> smallest) is committed.
// Only the per-restart (geom, valid) word and torsion indices leave the kernel.
//
// k_select_batched — select_poses (heavy-atom RMSD in f64) over poses REPLAYED from the argmax keys
// and the committed torsion indices into shared-memory slots (no pose ever goes to device memory:
// 14 KB less DRAM traffic per ligand and no N x atoms scratch), and an integer fixed-point rescore
// (order-free, exact) with pocket atoms (negated-coordinate f32x2 pairs, two per lane), weights and
// the bin look-up table staged in shared memory.
#include "ds_kernels.cuh"

namespace ds {

constexpr int kMaxA = DS_MAX_ATOMS;  // atom stride of the global final-pose scratch
constexpr int kInline = 3;           // bump candidates kept inline per moving atom
constexpr int kOvf = 32;             // per-fragment overflow list of further (moving, candidate) pairs
constexpr int kOptWarps = 8;         // warps per CTA of the select kernel (one ligand each)
constexpr int kTorWarps = 8;         // warps per CTA of the torsion kernel (1-warp CTAs measured slower)
#ifndef DS_SEL_MIN_BLOCKS
#define DS_SEL_MIN_BLOCKS 4          // select: 4 x 8 warps resident (<= 64 registers)
#endif
#ifndef DS_OPT_MIN_BLOCKS
#define DS_OPT_MIN_BLOCKS 4          // resident CTAs per SM the register budget is sized for
#endif

// Per-warp shared scratch of the torsion kernel (34 KB per 8-warp CTA at MA = 160, 28 KB at 128,
// 15 KB at 64: 4 CTAs per SM, registers bind; the rest of the SM's L1/shared array caches the grid
// gathers, so the launch takes the smallest MA that holds its largest ligand).
template <int MA>  // MA: the largest ligand the launch may hold (a multiple of 32, <= kMaxA)
struct TorWarpSmem {
  float4 u[MA];          // committed pose of the current restart (grid frame), .w: see mlist
  // moving atoms of the current fragment, ascending: their indices into u (a sweep lane takes slots
  // 2j, 2j+1 and packs their coordinates into f32x2 pairs); a moving atom's u[i].w holds its info
  // word for the fragment: bits 0-7 bump-candidate count, 8-15 / 16-23 / 24-31 the first three
  // candidates
  uint8_t mlist[MA];
  // cylindrical (h, r) as two arrays (C' pairs load as f32x2): C' atoms in [0, nCf) (+ one far pad
  // entry), moving atom m at MA-1-m
  f2_t chh2[MA / 2], chr2[MA / 2];
  uint8_t clist[MA];     // complement atom indices, ascending
  uint16_t ovf[kOvf];       // candidates beyond kInline: moving slot << 8 | atom index
  int n_ovf;                // entries appended (> kOvf: the list overflowed, scan C')
  int mhit[32];             // early exit: per sweep lane, the moving slot of its bump (P14 row count)
};

// Per-warp header of the select/rescore kernel's scratch; two pose slots of slot_atoms float4 follow
// (the candidate being replayed and a kept pose replayed for an exact RMSD; .w = the atom's
// weight-table row offset); cen[DS_MAX_RESTARTS] is the second slot's centroid scratch
struct SelHdr {
  double cen[DS_MAX_RESTARTS + 1][3];  // heavy-atom coordinate sums of the slots (RMSD lower bound)
  int geom[DS_MAX_RESTARTS];
  uint8_t valid[DS_MAX_RESTARTS];
  uint8_t ord[DS_MAX_RESTARTS];
  uint8_t kept[DS_MAX_RESTARTS];
};

__device__ __forceinline__ int grid_val(const PocketView &pk, int idx) { return (int)__ldg(pk.grid + idx) - 128; }

__device__ __forceinline__ int warp_sum(int v) { return (int)__reduce_add_sync(kFull, (unsigned)v); }

__device__ __forceinline__ long long warp_sum64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// cylindrical coordinates (h along the axis, r from it) of p about the axis through a along k;
// only used for the conservative culling bound (0.02-node margin), so its rounding does not matter:
// the hardware square-root approximation (relative error ~2^-22, < 1e-4 nodes here) instead of the
// IEEE sequence of the numeric recipe
__device__ __forceinline__ float2 cyl_coords(float4 p, float3 a, float kx, float ky, float kz) {
  const float wx = p.x - a.x, wy = p.y - a.y, wz = p.z - a.z;
  const float h = wx * kx + wy * ky + wz * kz;
  const float r2 = fmaxf(wx * wx + wy * wy + wz * wz - h * h, 0.f);
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(r2));
  return make_float2(h, r);
}

// order-preserving float <-> int map (an involution), so warp min/max reductions run on REDUX
__device__ __forceinline__ int ordered_bits(float f) {
  const int b = __float_as_int(f);
  return b ^ ((b >> 31) & 0x7FFFFFFF);
}
__device__ __forceinline__ float from_ordered_bits(int b) { return __int_as_float(b ^ ((b >> 31) & 0x7FFFFFFF)); }

// rotated position of a moving atom for torsion angle index k (k == 0: identity, P8)
__device__ __forceinline__ float3 torsion_pos(const PocketView &pk, int step_t, int k, float kx, float ky, float kz,
                                              float3 a, float4 p) {
  if (k == 0) return make_float3(p.x, p.y, p.z);
  const float2 cs = pk.trig[k * step_t];
  float R[9];
  torsion_matrix(kx, ky, kz, cs.x, cs.y, R);
  return torsion_apply(R, a, p.x, p.y, p.z);
}

// Packed rescore (P11): each lane owns TWO pocket atoms (j and j + 32 of a 64-atom round), staged
// in shared memory as negated-coordinate pairs, so the squared distances of a ligand atom to both
// come from FADD2 / FMUL2 / FFMA2 (each half bit-identical to dist2: x - y == x + (-y) exactly).
// The ligand atom (broadcast) is loaded once for the two pairs.  Bin: LUT or compares.
template <int kLut, typename Part>  // kLut: 0 compares, 1 clamped table, 2 full-range table
__device__ __forceinline__ long long rescore_pose_x2(const float4 *su, int A, const f2_t *pnx, const f2_t *pny,
                                                     const f2_t *pnz, const int2 *pcol, int nrounds,
                                                     const int32_t *wfx, int nb, const float *ub2,
                                                     const uint8_t *lut, int lut_shift, int lut_cap,
                                                     int part_atoms) {
  const int lane = threadIdx.x & 31;
  long long acc = 0;
  for (int k = 0; k < nrounds; ++k) {
    const f2_t NX = pnx[k * 32 + lane], NY = pny[k * 32 + lane], NZ = pnz[k * 32 + lane];
    const int2 col = pcol[k * 32 + lane];
    // int32 partials over part_atoms ligand atoms (2 terms each), which the host sized so that no
    // partial can overflow (PocketView::part_terms); widened to int64 between chunks
    for (int i0 = 0; i0 < A; i0 += part_atoms) {
      Part part = 0;
      const int i1 = min(A, i0 + part_atoms);
      for (int i = i0; i < i1; ++i) {
        const float4 x = su[i];
        const f2_t DX = f2_add(f2_pack(x.x, x.x), NX);
        const f2_t DY = f2_add(f2_pack(x.y, x.y), NY);
        const f2_t DZ = f2_add(f2_pack(x.z, x.z), NZ);
        float d0, d1;
        f2_unpack(f2_fma(DZ, DZ, f2_fma(DY, DY, f2_mul(DX, DX))), d0, d1);
        int b0 = __float_as_int(x.w) + col.x, b1 = __float_as_int(x.w) + col.y;  // .w: the row offset
        if (kLut == 2) {  // d2 >= +0: bits >> shift <= lut_cap by construction
          b0 += lut[(unsigned)__float_as_int(d0) >> lut_shift];
          b1 += lut[(unsigned)__float_as_int(d1) >> lut_shift];
        } else if (kLut == 1) {
          b0 += lut[min((unsigned)__float_as_int(d0) >> lut_shift, (unsigned)lut_cap)];
          b1 += lut[min((unsigned)__float_as_int(d1) >> lut_shift, (unsigned)lut_cap)];
        } else {
          for (int q = 0; q < nb; ++q) {
            b0 += !(d0 < ub2[q]);
            b1 += !(d1 < ub2[q]);
          }
        }
        part += (Part)wfx[b0] + (Part)wfx[b1];
      }
      acc += part;
    }
  }
  return acc;
}

// Replay restart r of ligand lig into P (grid frame, .w = weight-table row offset): the aligned
// pose from the argmax key (P6), then every committed torsion in fragment order (P8) with the axis
// taken from the current positions — the torsion kernel's operations, so the same bits.  Returns the
// heavy-atom coordinate sums (f64, any order: only used as a bound) in cen.
__device__ __forceinline__ void replay_pose(float4 *P, double *cen, const PocketView &pk, const BatchView &bt,
                                            const DockParams &dp, const uint32_t *keys, const OptOut &out, int lig,
                                            int r, int a0, int A, int f0, int F, int rowmul) {
  const int lane = threadIdx.x & 31;
  const unsigned key = keys[(size_t)lig * dp.N + r];
  const int rot = 65535 - (int)(key & 0xFFFFu);
  const int ix = rot / dp.n_a, iy = rot - ix * dp.n_a;
  {
    float R0s[9], T[3], Rp[9];
    start_params(bt.idh[lig], dp.seed, r, pk.trig, pk.inv_s, pk.g.nx, pk.g.ny, pk.g.nz, R0s, T);
    align_rx(pk.trig[ix * dp.step_a], R0s, Rp);
    const float2 cy = pk.trig[iy * dp.step_a];
    for (int i = lane; i < A; i += 32) {
      const float4 d = __ldg(bt.atoms + a0 + i);
      const float3 u = align_u(align_v(Rp, d.x, d.y, d.z), cy.x, cy.y, T);
      P[i] = make_float4(u.x, u.y, u.z, __int_as_float((int)d.w * rowmul));
    }
  }
  __syncwarp();
  for (int f = 0; f < F; ++f) {
    const int k = out.rtors[(size_t)(f0 + f) * dp.N + r];
    if (k == 0 || k == DS_TORSION_NONE) continue;  // angle 0 / all bumped: positions unchanged
    const uint4 fa = __ldg(bt.frags + 2 * (size_t)(f0 + f));
    const uint4 fb = __ldg(bt.frags + 2 * (size_t)(f0 + f) + 1);
    const unsigned mw[5] = {fa.x, fa.y, fa.z, fa.w, fb.x};
    const int ab = (int)(fb.y & 0xFFu), ae = (int)((fb.y >> 8) & 0xFFu);
    const float4 pa = P[ab], pb = P[ae];
    const float vx = __fsub_rn(pb.x, pa.x), vy = __fsub_rn(pb.y, pa.y), vz = __fsub_rn(pb.z, pa.z);
    const float len = __fsqrt_rn(__fmaf_rn(vz, vz, __fmaf_rn(vy, vy, __fmul_rn(vx, vx))));
    const float kx = __fdiv_rn(vx, len), ky = __fdiv_rn(vy, len), kz = __fdiv_rn(vz, len);
    const float3 a3 = make_float3(pa.x, pa.y, pa.z);
    for (int i = lane; i < A; i += 32)
      if ((mw[i >> 5] >> (i & 31)) & 1u) {  // axis atoms are never in the mask: read before any write
        const float4 p = P[i];
        const float3 q = torsion_pos(pk, dp.step_t, k, kx, ky, kz, a3, p);
        P[i] = make_float4(q.x, q.y, q.z, p.w);
      }
    __syncwarp();
  }
  double sx = 0.0, sy = 0.0, sz = 0.0;
  for (int i = lane; i < A; i += 32) {
    const float4 p = P[i];
    if (__float_as_int(p.w) != 0) {
      sx += (double)p.x;
      sy += (double)p.y;
      sz += (double)p.z;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sx += __shfl_xor_sync(kFull, sx, o);
    sy += __shfl_xor_sync(kFull, sy, o);
    sz += __shfl_xor_sync(kFull, sz, o);
  }
  if (lane == 0) {
    cen[0] = sx;
    cen[1] = sy;
    cen[2] = sz;
  }
  __syncwarp();
}

// P12 for one pair of poses: heavy-atom sum of squared deltas in f64 in atom order (the oracle's
// order), keep iff H > 0 and sum >= thr2 * H.  Returns true iff the poses are dissimilar.
__device__ __noinline__ bool pose_pair_dissimilar(const float4 *up, const float4 *uq, int A, int heavy, double thr2) {
  double sum = 0.0;
  for (int i = 0; i < A; ++i) {
    const float4 x = up[i], y = uq[i];
    if (__float_as_int(x.w) == 0) continue;
    const double dx = __dsub_rn((double)x.x, (double)y.x);
    const double dy = __dsub_rn((double)x.y, (double)y.y);
    const double dz = __dsub_rn((double)x.z, (double)y.z);
    double t = __dmul_rn(dx, dx);
    t = __dadd_rn(t, __dmul_rn(dy, dy));
    t = __dadd_rn(t, __dmul_rn(dz, dz));
    sum = __dadd_rn(sum, t);
  }
  return heavy > 0 && sum >= __dmul_rn(thr2, (double)heavy);
}

// minimum squared distance from q to the bump candidates of moving slot m beyond the inline ones:
// the fragment's overflow list, or every prefiltered C' atom when that list overflowed (cold path)
template <typename SM>
__device__ __forceinline__ float overflow_min(const SM &S, int m, int n_ovf, int nCf, float3 q) {
  float mind = __int_as_float(0x7f800000);
  if (n_ovf <= kOvf) {
#pragma unroll 1
    for (int t = 0; t < n_ovf; ++t) {
      const unsigned e = S.ovf[t];
      if ((int)(e >> 8) == m) {
        const float4 y = S.u[e & 0xFFu];
        mind = fminf(mind, dist2(q.x, q.y, q.z, y.x, y.y, y.z));
      }
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < nCf; ++c) {
      const float4 y = S.u[S.clist[c]];
      mind = fminf(mind, dist2(q.x, q.y, q.z, y.x, y.y, y.z));
    }
  }
  return mind;
}

// P9 bump test of a rotated moving atom q against its candidates (info word of its record):
// true iff some candidate lies strictly closer than the bump distance
template <typename SM>
__device__ __forceinline__ bool bump_hit(const SM &S, unsigned info, float3 q, int m, int n_ovf, int nCf,
                                         float bd2) {
  const unsigned cnt = info & 0xFFu;
  if (cnt == 0u) return false;
  const float4 y0 = S.u[(info >> 8) & 0xFFu];
  float mind = dist2(q.x, q.y, q.z, y0.x, y0.y, y0.z);  // min squared distance
  if (cnt > 1u) {
    const float4 y1 = S.u[(info >> 16) & 0xFFu];
    mind = fminf(mind, dist2(q.x, q.y, q.z, y1.x, y1.y, y1.z));
    if (cnt > 2u) {
      const float4 y2 = S.u[info >> 24];
      mind = fminf(mind, dist2(q.x, q.y, q.z, y2.x, y2.y, y2.z));
      if (cnt > (unsigned)kInline) mind = fminf(mind, overflow_min(S, m, n_ovf, nCf, q));
    }
  }
  return mind < bd2;
}

// A DegenerateAxis stops the ligand where the sequential oracle stops: restart records from the
// stopping restart on and torsion indices of (restart rd, fragments >= fd) and of later restarts
// are left zero, as the oracle leaves them (warp-cooperative, cold path)
__device__ __noinline__ void clear_unreached(const OptOut &out, int N, int f0, int F, int rd, int fd, int lig) {
  const int lane = threadIdx.x & 31;
  if (out.rrec)
    for (int r = rd + lane; r < N; r += 32) {
      ds_restart_record z;
      memset(&z, 0, sizeof z);
      out.rrec[(size_t)lig * N + r] = z;
    }
  for (int q = lane; q < F * N; q += 32) {
    const int f = q / N, r = q - f * N;
    if (r > rd || (r == rd && f >= fd)) out.rtors[(size_t)(f0 + f) * N + r] = 0;
  }
}

// kEarly: DockConfig.early_exit; kNT: the torsion angle count when it is the default
// 10 (torsion_step_deg = 36: the sweep's lane layout and loops become constants), 0 = runtime
template <bool kEarly, int kNT, int MA>
__global__ void __launch_bounds__(kTorWarps * 32, DS_OPT_MIN_BLOCKS)
    k_torsion_batched(PocketView pk, BatchView bt, DockParams dp, const int *order, const uint32_t *keys,
                      OptOut out, int *queue) {
  // per-warp scratch at a compile-time offset of the shared window (nothing to rematerialise from
  // launch parameters); dynamic because it exceeds the 48 KB static limit
  extern __shared__ __align__(16) unsigned char s_tor[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  TorWarpSmem<MA> &S = reinterpret_cast<TorWarpSmem<MA> *>(s_tor)[warp];
  const GridGeom g = pk.g;
  const unsigned lt = lanemask_lt();

  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(queue, 1);
    item = __shfl_sync(kFull, item, 0);
    if (item >= bt.L) break;
    const int lig = order ? order[item] : item;
    const int a0 = bt.atom_off[lig];
    const int A = bt.atom_off[lig + 1] - a0;
    const int f0 = bt.frag_off[lig];
    const int F = bt.frag_off[lig + 1] - f0;
    const uint64_t idh = bt.idh[lig];
    unsigned pairs_total = 0, early_exits = 0, evals = 0;
    bool degenerate = false;
    int n_aligned = dp.N;  // restarts whose alignment counts (P14; all unless a DegenerateAxis stops early)
    int deg_f = 0;         // the fragment that stopped it

    for (int r = 0; r < dp.N && !degenerate; ++r) {
      // ---- rebuild the aligned pose from the argmax key (P6) ----
      const unsigned key = keys[(size_t)lig * dp.N + r];
      const int rot = 65535 - (int)(key & 0xFFFFu);
      const int align_score = (int)(key >> 16) - 32768;
      // grid score of the current pose, carried along the fragment chain: the aligned pose scores
      // align_score (the key), a committed angle scores its key; a fragment's non-moving atoms then
      // score total - (its moving atoms at angle 0), so no per-fragment pass over them
      int total = align_score;
      const int ix = rot / dp.n_a, iy = rot - ix * dp.n_a;
      {
        float R0s[9], T[3], Rp[9];
        start_params(idh, dp.seed, r, pk.trig, pk.inv_s, g.nx, g.ny, g.nz, R0s, T);
        align_rx(pk.trig[ix * dp.step_a], R0s, Rp);
        const float2 cy = pk.trig[iy * dp.step_a];
        for (int i = lane; i < A; i += 32) {
          const float4 d = __ldg(bt.atoms + a0 + i);
          const float3 u = align_u(align_v(Rp, d.x, d.y, d.z), cy.x, cy.y, T);
          S.u[i] = make_float4(u.x, u.y, u.z, d.w);
        }
      }
      __syncwarp();

      // ---- optimize_pose: fragments in list order (P7-P10) ----
      int all_bumped = 0;
      for (int f = 0; f < F; ++f) {
        const uint4 fa = __ldg(bt.frags + 2 * (size_t)(f0 + f));
        const uint4 fb = __ldg(bt.frags + 2 * (size_t)(f0 + f) + 1);
        const unsigned mw5[5] = {fa.x, fa.y, fa.z, fa.w, fb.x};
        const int ab = (int)(fb.y & 0xFFu), ae = (int)((fb.y >> 8) & 0xFFu);
        // compaction of the moving set M (positions into mw) and of the bump-relevant complement C'
        // (not M, not an axis atom); base = grid score of the atoms the torsion does not move
        int nM = 0, nC = 0;
#pragma unroll
        for (int s = 0; s < 5; ++s) {
          if (s * 32 >= A) break;
          const int i = s * 32 + lane;
          const bool in = i < A;
          const bool mv = in && ((mw5[s] >> lane) & 1u);
          const bool cp = in && !mv && i != ab && i != ae;
          const unsigned bm = __ballot_sync(kFull, mv), bc = __ballot_sync(kFull, cp);
          if (mv) S.mlist[nM + __popc(bm & lt)] = (uint8_t)i;
          if (cp) S.clist[nC + __popc(bc & lt)] = (uint8_t)i;
          nM += __popc(bm);
          nC += __popc(bc);
        }
        int base = 0;  // score of the atoms the torsion does not move: total - angle-0 sum over M
        const float4 pa = S.u[ab], pb = S.u[ae];
        const float3 a3 = make_float3(pa.x, pa.y, pa.z);
        float kx = 0.f, ky = 0.f, kz = 0.f;
        if (kNT > 1 || (kNT == 0 && dp.n_t > 1)) {
          const float vx = __fsub_rn(pb.x, pa.x), vy = __fsub_rn(pb.y, pa.y), vz = __fsub_rn(pb.z, pa.z);
          const float len = __fsqrt_rn(__fmaf_rn(vz, vz, __fmaf_rn(vy, vy, __fmul_rn(vx, vx))));
          if (!(len >= dp.eps_axis)) {  // DegenerateAxis
            degenerate = true;
            deg_f = f;
            break;
          }
          kx = __fdiv_rn(vx, len);
          ky = __fdiv_rn(vy, len);
          kz = __fdiv_rn(vz, len);
        }
        __syncwarp();
        // ---- bump candidates per moving atom: cylindrical coordinates of C' in chr[0, nC) and of M
        // in chr[MA-1-m] (nM + nC <= A - 2), then every (m, c) pair tested by a flat lane loop;
        // survivors are counted into the moving atom's info word, the first kInline of them are kept
        // inline and the rest go to a short per-fragment overflow list (their order is irrelevant:
        // only the minimum distance is used).
        // The (h, r) box of M grown by the culling radius prefilters C': an atom outside it is
        // farther than the radius from every moving atom's circle, so it can never bump and is
        // dropped from the pair loop and the overflow scan (nCf <= nC; the P14 counters still count
        // all nC complement atoms).
        int hlo = 0x7FFFFFFF, hhi = (int)0x80000000, rhi = 0;
        if (lane == 0) S.n_ovf = 0;
        for (int m = lane; m < nM; m += 32) {
          const float4 pm = S.u[S.mlist[m]];
          const float2 hr = cyl_coords(pm, a3, kx, ky, kz);
          reinterpret_cast<float *>(S.chh2)[MA - 1 - m] = hr.x;
          reinterpret_cast<float *>(S.chr2)[MA - 1 - m] = hr.y;
          hlo = min(hlo, ordered_bits(hr.x));
          hhi = max(hhi, ordered_bits(hr.x));
          rhi = max(rhi, __float_as_int(hr.y));  // r >= +0: bit order is float order
        }
        const float cut = dp.cull_r;
        const float h0 = __fsub_rn(from_ordered_bits(__reduce_min_sync(kFull, hlo)), cut);
        const float h1 = __fadd_rn(from_ordered_bits(__reduce_max_sync(kFull, hhi)), cut);
        const float r1 = __fadd_rn(__int_as_float(__reduce_max_sync(kFull, rhi)), cut);
        int nCf = 0;
        for (int c0 = 0; c0 < nC; c0 += 32) {
          const int c = c0 + lane;
          float2 hr = make_float2(0.f, 0.f);
          uint8_t ci = 0;
          bool keep = false;
          if (c < nC) {
            ci = S.clist[c];
            hr = cyl_coords(S.u[ci], a3, kx, ky, kz);
            keep = hr.x > h0 && hr.x < h1 && hr.y < r1;
          }
          const unsigned bk = __ballot_sync(kFull, keep);  // in-place compaction: slot <= c
          __syncwarp();  // every lane's read of clist[c] is ordered before the overwrites
          if (keep) {
            const int slot = nCf + __popc(bk & lt);
            reinterpret_cast<float *>(S.chh2)[slot] = hr.x;
            reinterpret_cast<float *>(S.chr2)[slot] = hr.y;
            S.clist[slot] = ci;
          }
          nCf += __popc(bk);
        }
        // far pad after the last C' entry (slot nCf < MA - nM since nCf + nM <= A - 2): an odd
        // nCf still tests whole f32x2 pairs and the pad never passes the bound
        if (lane == 0) {
          reinterpret_cast<float *>(S.chh2)[nCf] = 3.0e38f;
          reinterpret_cast<float *>(S.chr2)[nCf] = 3.0e38f;
        }
        __syncwarp();
        // lane = moving atom, loop over the prefiltered C' (broadcast reads): the lane owns its info
        // word, so candidates are recorded without shared atomics (only the rare overflow appends)
        for (int m0 = 0; m0 < nM; m0 += 32) {
          const int m = m0 + lane;
          const bool ok = m < nM;
          const float hmh = ok ? reinterpret_cast<const float *>(S.chh2)[MA - 1 - m] : 3.0e38f;
          const float hmr = ok ? reinterpret_cast<const float *>(S.chr2)[MA - 1 - m] : 3.0e38f;
          const f2_t HM = f2_pack(hmh, hmh), RM = f2_pack(hmr, hmr);
          unsigned cnt = 0, inl = 0;
          // two C' atoms per iteration with packed f32x2 (the bound is conservative, so any rounding
          // of this test is fine)
          for (int c = 0; c < nCf; c += 2) {
            const f2_t DH = f2_sub(HM, S.chh2[c >> 1]), DR = f2_sub(RM, S.chr2[c >> 1]);
            float d0, d1;
            f2_unpack(f2_fma(DH, DH, f2_mul(DR, DR)), d0, d1);
            const bool k0 = d0 < dp.cull2, k1 = d1 < dp.cull2;
            if (k0 || k1) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                if (!(h ? k1 : k0)) continue;
                const unsigned ci = S.clist[c + h];
                if (cnt < (unsigned)kInline) {
                  inl |= ci << (8 + 8 * cnt);
                } else {
                  const int slot = atomicAdd(&S.n_ovf, 1);
                  if (slot < kOvf) S.ovf[slot] = (uint16_t)((m << 8) | ci);
                }
                ++cnt;
              }
            }
          }
          // the info word rides in the moving atom's .w (unused by the torsion kernel otherwise), so
          // the sweep gets it with the atom's position load
          if (ok) reinterpret_cast<unsigned *>(&S.u[S.mlist[m]])[3] = cnt | inl;  // cnt <= nCf < 256
        }
        unsigned best_key = 0;  // (score + 32768) << 16 | (65535 - angle); 0 = no clean angle
        __syncwarp();
        const int n_ovf = S.n_ovf;
        // ---- all angles at once: lane = (angle a, moving-atom group gi); the lane keeps its angle's
        // rotation, bump flag and partial score in registers over moving atoms m = gi, gi+G, ...
        // Angle 0 (the identity, P7) runs the same code with R = I about the origin: w = p - 0 = p and
        // fma(0, ., fma(0, ., fma(1, p, 0))) = p up to the sign of a zero, which changes neither a
        // node nor a squared distance (and angle 0 is never committed).
        const int n_t = kNT ? kNT : dp.n_t;
        for (int k0 = 0; k0 < n_t; k0 += 32) {
          const int nA = kNT ? kNT : min(32, n_t - k0);
          int G, a, gi;                           // moving-atom groups per round, lane's angle and group
          unsigned same;                          // lanes that share this lane's angle
          if (kNT) {                              // compile-time layout: lane = gi * kNT + a
            G = 32 / kNT;
            a = lane % kNT;
            gi = lane / kNT;
            same = 0;
#pragma unroll
            for (int t = 0; t < 32 / kNT; ++t) same |= 1u << (a + t * kNT);
          } else if (k0 == 0) {                   // host-built layout of the first block
            const unsigned e = dp.sweep_lane[lane];
            a = (int)(e & 0xFFu);
            gi = (int)((e >> 8) & 0xFFu);
            same = dp.sweep_same[lane];
            G = __popc(dp.sweep_same[0]);
          } else {
            G = 32 / nA;
            a = lane % nA;
            gi = lane / nA;
            same = 0;
            for (int t = 0; t < G; ++t) same |= 1u << (a + t * nA);
          }
          const bool lane_ok = gi < G;
          const int kang = k0 + a;
          float R[9] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f, 1.f};
          float3 ar = make_float3(0.f, 0.f, 0.f);
          if (kang > 0) {
            const float2 cs = pk.trig[kang * (kNT ? 360 / kNT : dp.step_t)];
            torsion_matrix(kx, ky, kz, cs.x, cs.y, R);
            ar = a3;
          }
          bool bumped = false;
          int part = 0;
          S.mhit[lane] = 0x7FFFFFFF;
          // two moving atoms per lane and round (slots m0 + 2 gi and m0 + 2 gi + 1): twice the
          // independent work (two grid loads in flight) for the same loop and retirement overhead,
          // and the two rotations run as packed f32x2 (FADD2 / FFMA2, each half the scalar recipe)
          const f2_t R0 = f2_pack(R[0], R[0]), R1 = f2_pack(R[1], R[1]), R2 = f2_pack(R[2], R[2]);
          const f2_t R3 = f2_pack(R[3], R[3]), R4 = f2_pack(R[4], R[4]), R5 = f2_pack(R[5], R[5]);
          const f2_t R6 = f2_pack(R[6], R[6]), R7 = f2_pack(R[7], R[7]), R8 = f2_pack(R[8], R[8]);
          const f2_t AX = f2_pack(ar.x, ar.x), AY = f2_pack(ar.y, ar.y), AZ = f2_pack(ar.z, ar.z);
          const f2_t NAX = f2_pack(-ar.x, -ar.x), NAY = f2_pack(-ar.y, -ar.y), NAZ = f2_pack(-ar.z, -ar.z);
          const f2_t MM = f2_pack(kMagic, kMagic);
          for (int m0 = 0; m0 < nM; m0 += 2 * G) {
            const int m1 = m0 + 2 * gi, m2 = m1 + 1;
            // with early exit a bumped angle is retired; without it every pair is checked
            // angle 0 is never retired: its complete sum gives the non-moving atoms' score
            const bool live = lane_ok && !(kEarly && bumped && kang != 0);
            const bool act1 = live && m1 < nM, act2 = live && m2 < nM;
            if (!__any_sync(kFull, act1)) break;
            bool hit = false;
            if (act1) {
              const int j = m1 >> 1;
              // w = p - a (as p + (-a): exact negation), p' = R w + a (P8), then + magic (P4)
              const float4 p1 = S.u[S.mlist[m1]], p2 = S.u[S.mlist[act2 ? m2 : m1]];
              const f2_t WX = f2_add(f2_pack(p1.x, p2.x), NAX), WY = f2_add(f2_pack(p1.y, p2.y), NAY),
                         WZ = f2_add(f2_pack(p1.z, p2.z), NAZ);
              const f2_t QX = f2_fma(R2, WZ, f2_fma(R1, WY, f2_fma(R0, WX, AX)));
              const f2_t QY = f2_fma(R5, WZ, f2_fma(R4, WY, f2_fma(R3, WX, AY)));
              const f2_t QZ = f2_fma(R8, WZ, f2_fma(R7, WY, f2_fma(R6, WX, AZ)));
              float mx1, mx2, my1, my2, mz1, mz2;
              f2_unpack(f2_add(QX, MM), mx1, mx2);
              f2_unpack(f2_add(QY, MM), my1, my2);
              f2_unpack(f2_add(QZ, MM), mz1, mz2);
              // both grid loads are issued before the candidate checks: they hide each other's latency
              const int gv1 = grid_val(pk, node_index_magic(g, mx1, my1, mz1));
              const int gv2 = grid_val(pk, node_index_magic(g, mx2, my2, mz2));
              float3 q1, q2;
              f2_unpack(QX, q1.x, q2.x);
              f2_unpack(QY, q1.y, q2.y);
              f2_unpack(QZ, q1.z, q2.z);
              const uint2 info = make_uint2(__float_as_uint(p1.w), __float_as_uint(p2.w));
              const bool h1 = bump_hit(S, info.x, q1, m1, n_ovf, nCf, dp.bd2);
              const bool h2 = act2 && bump_hit(S, info.y, q2, m2, n_ovf, nCf, dp.bd2);
              part += gv1 + (act2 ? gv2 : 0);  // a bumped angle's sum is never used
              hit = h1 || h2;
              // with early exit an angle bumps in one round only (it is retired after it)
              if (kEarly && hit && !bumped) S.mhit[lane] = h1 ? m1 : m2;
            }
            if (kEarly) {  // OR the hits of the G lanes that share an angle
              // every lane must reach the ballot: never put it behind a short-circuit operator
              const unsigned hb = __ballot_sync(kFull, hit);
              bumped = bumped || (hb & same) != 0u;
            } else {
              bumped = bumped || hit;
            }
          }
          __syncwarp();
          // pairs evaluated at moving-row granularity (P14): all nM * nC of a clean angle (or without
          // early exit), else the whole rows of the moving slots up to and including the first
          // bumping one, m* = the smallest bumping slot of the angle's G lanes
          {
            unsigned np = 0;
            if (gi == 0 && lane_ok) {
              int mb = 0x7FFFFFFF;
              for (int t = 0; t < G; ++t) mb = min(mb, S.mhit[a + t * nA]);
              np = mb == 0x7FFFFFFF ? (unsigned)(nM * nC) : (unsigned)((mb + 1) * nC);
            }
            pairs_total += (unsigned)warp_sum((int)np);
          }
          __syncwarp();
          // combine the G partial scores of an angle on its group-0 lane
          int sum = part;
          for (int t = 1; t < G; ++t) {
            const int v = __shfl_down_sync(kFull, part, t * nA);
            if (gi == 0) sum += v;
          }
          if (k0 == 0) base = total - __shfl_sync(kFull, sum, 0);  // lane 0: angle 0, group 0
          unsigned hb = __ballot_sync(kFull, bumped && lane_ok);
          unsigned fold = 0;
          for (int t = 0; t < G; ++t) fold |= hb >> (t * nA);
          fold &= nA == 32 ? 0xFFFFFFFFu : ((1u << nA) - 1u);
          unsigned kk = 0;
          if (gi == 0 && !((fold >> a) & 1u))
            kk = ((unsigned)(base + sum + 32768) << 16) | (unsigned)(65535 - kang);
          evals += (unsigned)nA;
          if (kEarly) early_exits += (unsigned)__popc(fold);
          best_key = max(best_key, __reduce_max_sync(kFull, kk));
        }
        const int best_k = best_key ? 65535 - (int)(best_key & 0xFFFFu) : -1;
        if (best_key) total = (int)(best_key >> 16) - 32768;  // the committed pose's score
        // commit the winner before the next fragment; moving slot m of atom i is its rank in the mask
        if (best_k > 0) {
          const uint4 ga = __ldg(bt.frags + 2 * (size_t)(f0 + f));
          const unsigned gm[5] = {ga.x, ga.y, ga.z, ga.w, __ldg(bt.frags + 2 * (size_t)(f0 + f) + 1).x};
          int mr = 0;
          for (int s = 0; s < 5 && s * 32 < A; ++s) {
            const int i = s * 32 + lane;
            const bool mv = i < A && ((gm[s] >> lane) & 1u);
            const unsigned bm = __ballot_sync(kFull, mv);
            if (mv) {
              const int m = mr + __popc(bm & lt);
              const float4 W = S.u[i];  // not yet moved: the committed pose's position
              const float3 q = torsion_pos(pk, kNT ? 360 / kNT : dp.step_t, best_k, kx, ky, kz, a3, W);
              S.u[i] = make_float4(q.x, q.y, q.z, S.u[i].w);
            }
            mr += __popc(bm);
          }
        }
        if (best_k < 0) ++all_bumped;
        if (lane == 0) out.rtors[(size_t)(f0 + f) * dp.N + r] = best_k < 0 ? (uint8_t)DS_TORSION_NONE : (uint8_t)best_k;
        __syncwarp();
      }
      if (degenerate) {  // the oracle stops the ligand here: restarts 0..r were aligned
        n_aligned = r + 1;
        break;
      }
      // final geometric score (carried); the select kernel replays the pose from the key and the
      // committed torsion indices, so no pose leaves the SM
      const int sc = total;
      const int valid = !(F >= 1 && all_bumped == F);  // P10
      if (lane == 0) {
        out.rgv[(size_t)lig * dp.N + r] = (sc * 2) | valid;
        if (out.rrec) {
          ds_restart_record rec;
          rec.align_score = align_score;
          rec.final_geom = sc;
          rec.ax = (uint8_t)ix;
          rec.ay = (uint8_t)iy;
          rec.valid = (uint8_t)valid;
          rec.kept = 0;
          rec.reserved = 0;
          out.rrec[(size_t)lig * dp.N + r] = rec;
        }
      }
      __syncwarp();
    }

    if (degenerate) clear_unreached(out, dp.N, f0, F, n_aligned - 1, deg_f, lig);
    // counters and the degenerate status; k_select_batched completes the record
    if (lane == 0) {
      ds_result res;
      res.geom_score = 0;
      res.chem_fx = 0;
      res.best_restart = 0;
      res.best_ax = 0;
      res.best_ay = 0;
      res.n_kept = 0;
      res.poses_scored = (unsigned)(n_aligned * dp.n_rot) + evals;
      res.bump_checks = pairs_total;
      res.bump_early_exits = early_exits;
      res.status = degenerate ? DS_STATUS_DEGENERATE_AXIS : DS_STATUS_OK;
      out.res[lig] = res;
    }
    __syncwarp();
  }
}

// Replay-based select_poses (P12) + rescore (P11).  Warp per ligand; the valid restarts are visited
// in (geom desc, restart asc) order and each is replayed into a free pose slot; the RMSD to every
// kept pose is first bounded below by the heavy-atom centroid distance (RMSD^2 >= |dc|^2 exactly,
// so a centroid distance beyond the threshold, with a 1e-6 relative margin that dwarfs the f64
// rounding of the sums, decides "dissimilar" exactly as the oracle's sum would), and only close
// pairs take the oracle's sequential f64 sum (one lane per kept pose).  The kept poses are then
// rescored from their slots.  Nothing is read back from device memory but the inputs, the keys,
// the torsion indices and the per-restart (geom, valid) words.
// kMode: the rescore's binning / accumulator (one instantiation each, chosen at launch from the
// pocket): 0 full-range bin table + int32 partials, 1 clamped table + int32, 2 compares + int32,
// 3 compares + int64 (tables whose weights do not fit two terms in an int32)
template <int kMode>
__global__ void __launch_bounds__(kOptWarps * 32, DS_SEL_MIN_BLOCKS)
    k_select_batched(PocketView pk, BatchView bt, DockParams dp, const uint32_t *keys, OptOut out, int *queue,
                     int tables_bytes, int warp_bytes) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // per-CTA: pocket atoms + fixed-point weights + bin bounds + bin LUT
  const int nb1 = pk.nb + 1;
  // pocket atoms as 64-atom rounds of lane pairs (j, j + 32): negated coordinates + weight columns
  const int nrounds = (pk.n_atoms + 63) / 64;
  f2_t *s_nx = reinterpret_cast<f2_t *>(smem);
  f2_t *s_ny = s_nx + nrounds * 32;
  f2_t *s_nz = s_ny + nrounds * 32;
  int2 *s_col = reinterpret_cast<int2 *>(s_nz + nrounds * 32);
  int32_t *s_w = reinterpret_cast<int32_t *>(s_col + nrounds * 32);
  const int wsz = DS_N_TYPES * DS_N_TYPES * nb1;
  float *s_ub2 = reinterpret_cast<float *>(s_w + wsz);
  uint8_t *s_lut = reinterpret_cast<uint8_t *>(s_ub2 + DS_MAX_BINS);
  for (int e = threadIdx.x; e < nrounds * 32; e += blockDim.x) {
    const int k = e >> 5, l = e & 31;
    float4 y[2];
    for (int h = 0; h < 2; ++h) {
      const int j = k * 64 + h * 32 + l;
      // past-the-end: a far sentinel, beyond every bin (weight column of type 0, entry nb -> 0)
      y[h] = j < pk.n_atoms ? __ldg(pk.patoms + j) : make_float4(1e19f, 1e19f, 1e19f, 0.f);
    }
    s_nx[e] = f2_pack(-y[0].x, -y[1].x);
    s_ny[e] = f2_pack(-y[0].y, -y[1].y);
    s_nz[e] = f2_pack(-y[0].z, -y[1].z);
    s_col[e] = make_int2((int)y[0].w * nb1, (int)y[1].w * nb1);
  }
  for (int j = threadIdx.x; j < wsz; j += blockDim.x) s_w[j] = __ldg(pk.wfx + j);
  if (threadIdx.x < DS_MAX_BINS) s_ub2[threadIdx.x] = pk.ub2[threadIdx.x];
  for (int j = threadIdx.x; j <= pk.lut_cap; j += blockDim.x) s_lut[j] = __ldg(pk.bin_lut + j);
  unsigned char *wbase = smem + tables_bytes + (size_t)warp * warp_bytes;
  SelHdr &S = *reinterpret_cast<SelHdr *>(wbase);
  float4 *slots = reinterpret_cast<float4 *>(wbase + ((sizeof(SelHdr) + 15) & ~(size_t)15));
  const int rowmul = DS_N_TYPES * nb1;
  // "dissimilar by the bound": |dc|^2 (in units of H^2: sums, not means) >= thr2 H^2 (1 + 1e-6)
  const double thr2_margin = __dmul_rn(dp.thr2, 1.000001);
  __syncthreads();

  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(queue, 1);
    item = __shfl_sync(kFull, item, 0);
    if (item >= bt.L) break;
    const int lig = out.sel_order ? out.sel_order[item] : item;
    ds_result res = out.res[lig];
    if (res.status != DS_STATUS_OK) continue;  // DegenerateAxis: already final
    const int a0 = bt.atom_off[lig];
    const int A = bt.atom_off[lig + 1] - a0;
    const int f0 = bt.frag_off[lig];
    const int F = bt.frag_off[lig + 1] - f0;
    // ---- select_poses (P12): order valid poses by (geom desc, restart asc) ----
    for (int r = lane; r < dp.N; r += 32) {
      const int gv = out.rgv[(size_t)lig * dp.N + r];
      S.geom[r] = gv >> 1;
      S.valid[r] = (uint8_t)(gv & 1);
    }
    int hv = 0;
    for (int i = lane; i < A; i += 32) hv += __ldg(bt.atoms + a0 + i).w != 0.f;
    const int heavy = warp_sum(hv);
    __syncwarp();
    int nvalid = 0;
    for (int r = 0; r < dp.N; ++r) nvalid += S.valid[r];
    if (nvalid == 0) {
      res.status = DS_STATUS_NO_VALID_POSE;
      if (lane == 0) out.res[lig] = res;
      __syncwarp();
      continue;
    }
    for (int r = lane; r < dp.N; r += 32) {
      if (S.valid[r]) {
        int rank = 0;
        for (int q = 0; q < dp.N; ++q)
          rank += S.valid[q] && (S.geom[q] > S.geom[r] || (S.geom[q] == S.geom[r] && q < r));
        S.ord[rank] = (uint8_t)r;
      }
    }
    __syncwarp();
    // greedy keep (warp-uniform): each candidate is replayed into the candidate slot; a kept pose
    // is rescored at once (and its coordinates written out while it is the best so far), so only
    // the kept poses' heavy-atom centroids stay — a kept pose the centroid bound cannot separate
    // from a later candidate (rare) is replayed again into the second slot for the exact sum
    const double hh = (double)heavy * (double)heavy;
    float4 *cand = slots, *xs = slots + dp.slot_atoms;
    int nk = 0;
    long long best_chem = 0;
    int best_r = -1;
    for (int o = 0; o < nvalid && nk < dp.K; ++o) {
      const int c = S.ord[o];
      replay_pose(cand, S.cen[nk], pk, bt, dp, keys, out, lig, c, a0, A, f0, F, rowmul);
      bool close = false;  // kept poses the bound cannot separate from the candidate
      if (lane < nk) {
        const double dx = S.cen[nk][0] - S.cen[lane][0], dy = S.cen[nk][1] - S.cen[lane][1],
                     dz = S.cen[nk][2] - S.cen[lane][2];
        close = !(heavy > 0 && dx * dx + dy * dy + dz * dz >= thr2_margin * hh);
      }
      unsigned cm = __ballot_sync(kFull, close);
      bool dis = true;
      while (cm && dis) {
        const int k = __ffs(cm) - 1;
        cm &= cm - 1;
        replay_pose(xs, S.cen[DS_MAX_RESTARTS], pk, bt, dp, keys, out, lig, S.kept[k], a0, A, f0, F, rowmul);
        int d = 1;
        if (lane == 0) d = pose_pair_dissimilar(cand, xs, A, heavy, dp.thr2);
        dis = __shfl_sync(kFull, d, 0) != 0;
      }
      if (!dis) continue;
      if (lane == 0) S.kept[nk] = (uint8_t)c;
      // ---- rescore the kept pose (P11): exact fixed-point sum over (ligand atom, pocket atom) ----
      // int32 partials when two weight terms fit (every default-like table), int64 otherwise
      long long acc;
      if (kMode == 0)
        acc = rescore_pose_x2<2, int>(cand, A, s_nx, s_ny, s_nz, s_col, nrounds, s_w, pk.nb, s_ub2, s_lut,
                                      pk.lut_shift, pk.lut_cap, pk.part_terms / 2);
      else if (kMode == 1)
        acc = rescore_pose_x2<1, int>(cand, A, s_nx, s_ny, s_nz, s_col, nrounds, s_w, pk.nb, s_ub2, s_lut,
                                      pk.lut_shift, pk.lut_cap, pk.part_terms / 2);
      else if (kMode == 2)
        acc = rescore_pose_x2<0, int>(cand, A, s_nx, s_ny, s_nz, s_col, nrounds, s_w, pk.nb, s_ub2, s_lut, 0, 0,
                                      pk.part_terms / 2);
      else
        acc = rescore_pose_x2<0, long long>(cand, A, s_nx, s_ny, s_nz, s_col, nrounds, s_w, pk.nb, s_ub2, s_lut, 0,
                                            0, A);
      acc = warp_sum64(acc);
      if (best_r < 0 || acc > best_chem || (acc == best_chem && c < best_r)) {
        best_chem = acc;
        best_r = c;
        if (out.best_coords)
          for (int i = lane; i < A; i += 32) {  // back to Å: q = fma(u, s, o)   (P2)
            const float4 x = cand[i];
            float *q = out.best_coords + 3 * (size_t)(a0 + i);
            q[0] = __fmaf_rn(x.x, pk.spacing, pk.ox);
            q[1] = __fmaf_rn(x.y, pk.spacing, pk.oy);
            q[2] = __fmaf_rn(x.z, pk.spacing, pk.oz);
          }
      }
      if (lane == 0 && out.rrec) out.rrec[(size_t)lig * dp.N + c].kept = (uint8_t)(nk + 1);
      ++nk;
      __syncwarp();
    }
    const unsigned bkey = keys[(size_t)lig * dp.N + best_r];
    const int brot = 65535 - (int)(bkey & 0xFFFFu);
    res.status = DS_STATUS_OK;
    res.geom_score = S.geom[best_r];
    res.chem_fx = best_chem;
    res.best_restart = (uint8_t)best_r;
    res.best_ax = (uint8_t)(brot / dp.n_a);
    res.best_ay = (uint8_t)(brot - (brot / dp.n_a) * dp.n_a);
    res.n_kept = (uint8_t)nk;
    if (lane == 0) out.res[lig] = res;
    if (out.best_tors)
      for (int f = lane; f < F; f += 32) out.best_tors[f0 + f] = out.rtors[(size_t)(f0 + f) * dp.N + best_r];
    __syncwarp();
  }
}

static size_t select_tables_bytes(int n_patoms, int nb, int lut_cap) {
  size_t fixed = (size_t)((n_patoms + 63) / 64) * 32 * 32 + (size_t)DS_N_TYPES * DS_N_TYPES * (nb + 1) * 4 +
                 DS_MAX_BINS * 4 + (size_t)(lut_cap + 1);
  return (fixed + 15) & ~(size_t)15;
}
static size_t select_warp_bytes(int K, int slot_atoms) {
  // two pose slots: the candidate and the on-demand replay of a kept pose (kept poses are rescored
  // when kept, so only their centroids stay)
  (void)K;
  return ((sizeof(SelHdr) + 15) & ~(size_t)15) + (size_t)2 * slot_atoms * sizeof(float4);
}
// dynamic shared memory of a k_select_batched CTA (kOptWarps warps) for top-K K and ligands of at
// most slot_atoms atoms
size_t select_cta_smem_bytes(int n_patoms, int nb, int lut_cap, int K, int slot_atoms) {
  return select_tables_bytes(n_patoms, nb, lut_cap) + kOptWarps * select_warp_bytes(K, slot_atoms);
}

template <int MA>
constexpr size_t tor_smem() { return kTorWarps * sizeof(TorWarpSmem<MA>); }

template <bool E, int NT, int MA>
static void launch_tors(const PocketView &pk, const BatchView &bt, const DockParams &dp, const int *order,
                        const uint32_t *keys, OptOut out, int *queue, int blocks, cudaStream_t st) {
  allow_max_smem((const void *)k_torsion_batched<E, NT, MA>);
  k_torsion_batched<E, NT, MA><<<blocks, kTorWarps * 32, tor_smem<MA>(), st>>>(pk, bt, dp, order, keys, out, queue);
}

// the scratch class of the launch: the smallest MA holding its largest ligand (dp.slot_atoms)
template <bool E, int NT>
static void launch_tors_ma(const PocketView &pk, const BatchView &bt, const DockParams &dp, const int *order,
                           const uint32_t *keys, OptOut out, int *queue, int blocks, cudaStream_t st) {
  if (NT && dp.slot_atoms <= 64) launch_tors<E, NT, 64>(pk, bt, dp, order, keys, out, queue, blocks, st);
  else if (NT && dp.slot_atoms <= 128) launch_tors<E, NT, 128>(pk, bt, dp, order, keys, out, queue, blocks, st);
  else launch_tors<E, NT, kMaxA>(pk, bt, dp, order, keys, out, queue, blocks, st);
}

void launch_torsion_batched(const PocketView &pk, const BatchView &bt, const DockParams &dp, const int *order,
                            const uint32_t *keys, OptOut out, int *queue, int blocks, cudaStream_t st) {
  const bool nt10 = dp.n_t == 10;
  if (dp.early_exit) {
    if (nt10) launch_tors_ma<true, 10>(pk, bt, dp, order, keys, out, queue, blocks, st);
    else launch_tors_ma<true, 0>(pk, bt, dp, order, keys, out, queue, blocks, st);
  } else {
    if (nt10) launch_tors_ma<false, 10>(pk, bt, dp, order, keys, out, queue, blocks, st);
    else launch_tors_ma<false, 0>(pk, bt, dp, order, keys, out, queue, blocks, st);
  }
}

// warps per CTA (1..kOptWarps) chosen for the most resident warps per SM: every CTA carries its
// own rescore tables beside its warps' pose slots (one warp always fits: 32 slots x 160 atoms x
// 16 B + the tables)
static int select_mode(const PocketView &pk) {
  if (pk.part_terms >= 2 && pk.lut_cap >= 0 && pk.lut_full) return 0;
  if (pk.part_terms >= 2 && pk.lut_cap >= 0) return 1;
  return pk.part_terms >= 2 ? 2 : 3;
}
static const void *select_kernel(int mode) {
  switch (mode) {
    case 0: return (const void *)k_select_batched<0>;
    case 1: return (const void *)k_select_batched<1>;
    case 2: return (const void *)k_select_batched<2>;
    default: return (const void *)k_select_batched<3>;
  }
}

void launch_select_batched(const PocketView &pk, const BatchView &bt, const DockParams &dp, const uint32_t *keys,
                           OptOut out, int *queue, int sm_count, size_t smem_optin, cudaStream_t st) {
  const int mode = select_mode(pk);
  const void *kern = select_kernel(mode);
  const size_t tb = select_tables_bytes(pk.n_atoms, pk.nb, pk.lut_cap), wb = select_warp_bytes(dp.K, dp.slot_atoms);
  int best_w = 1, best_res = 0, best_per_sm = 1;
  for (int w = 1; w <= kOptWarps; ++w) {
    const size_t smem = tb + w * wb;
    if (smem > smem_optin) break;
    allow_max_smem(kern);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, w * 32, smem);
    if (per_sm * w >= best_res) {
      best_res = per_sm * w;
      best_w = w;
      best_per_sm = std::max(1, per_sm);
    }
  }
  const size_t smem = tb + best_w * wb;
  allow_max_smem(kern);
  const int itb = (int)tb, iwb = (int)wb;
  void *args[] = {(void *)&pk, (void *)&bt, (void *)&dp, (void *)&keys, (void *)&out, (void *)&queue, (void *)&itb,
                  (void *)&iwb};
  cudaLaunchKernel(kern, dim3(sm_count * best_per_sm), dim3(best_w * 32), args, smem, st);
}

int torsion_blocks_per_sm() {
  int n = 0;
  allow_max_smem((const void *)k_torsion_batched<true, 10, kMaxA>);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_torsion_batched<true, 10, kMaxA>, kTorWarps * 32,
                                                tor_smem<kMaxA>());
  return n;
}

int select_blocks_per_sm(size_t smem) {
  int n = 0;
  allow_max_smem((const void *)k_select_batched<0>);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_select_batched<0>, kOptWarps * 32, smem);
  return n;
}

}  // namespace ds
