// Pose optimisation, pose selection and rescoring (Alg. 1 lines 10-21, PAPER.md:227-247;
// SPEC.md:257-285) — batched family, one warp per ligand.
//
// Per restart the warp rebuilds the aligned pose from the packed argmax key of the alignment
// kernel, then walks the fragments in list order.  Per fragment it compacts the moving set M and
// the bump-relevant complement C' (= not M, not an axis atom) into shared memory with ballots, and
// for every torsion angle rotates M, runs the M x C' bump scan in lexicographic pair order in
// rounds of 32 with a warp-uniform early exit (__any_sync — the zero-cost exit that makes the
// batched shape win), and scores clean angles as base + sum over M (the
// non-moving atoms' grid values do not change with the angle).  The best clean angle is
// committed before the next fragment.  Then select_poses (heavy-atom RMSD,
// f64, lanes over pose pairs) and an integer fixed-point rescore (order-free, exact).
#include "ds_kernels.cuh"

namespace ds {

constexpr int kMaxA = DS_MAX_ATOMS;

struct OptWarpSmem {
  float4 u[kMaxA];       // committed pose of the current restart (grid frame), .w = type
  float4 wk[kMaxA];      // [0, nM): moving atoms at the current angle; [kMaxA-1-c]: complement atom c
  uint8_t mlist[kMaxA];  // moving atom indices in ascending order
  int geom[DS_MAX_RESTARTS];
  int valid[DS_MAX_RESTARTS];
  unsigned dis[DS_MAX_RESTARTS];   // dissimilarity bitsets (select_poses)
  int ord[DS_MAX_RESTARTS];
  long long chem[DS_MAX_RESTARTS];
};

__device__ __forceinline__ int grid_val(const PocketView &pk, int idx) { return (int)__ldg(pk.grid + idx); }

__device__ __forceinline__ int warp_sum(int v) { return (int)__reduce_add_sync(kFull, (unsigned)v); }

__device__ __forceinline__ long long warp_sum64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__global__ void __launch_bounds__(256)
    k_optimize_batched(PocketView pk, BatchView bt, DockParams dp, const int *order, const uint32_t *keys,
                       OptOut out, int *queue) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  OptWarpSmem &S = reinterpret_cast<OptWarpSmem *>(smem)[warp];
  const int gwarp = blockIdx.x * (blockDim.x >> 5) + warp;
  float4 *scr = out.final_u + (size_t)gwarp * dp.N * kMaxA;  // final poses of the N restarts
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
    int heavy = 0;

    for (int r = 0; r < dp.N && !degenerate; ++r) {
      // ---- rebuild the aligned pose from the argmax key (P6) ----
      const unsigned key = keys[(size_t)lig * dp.N + r];
      const int rot = 65535 - (int)(key & 0xFFFFu);
      const int align_score = (int)(key >> 16) - 32768;
      const int ix = rot / dp.n_a, iy = rot - ix * dp.n_a;
      float R0s[9], T[3], M[9];
      start_params(idh, dp.seed, r, pk.trig, pk.inv_s, g.nx, g.ny, g.nz, R0s, T);
      align_matrix(pk.trig[ix * dp.step_a], pk.trig[iy * dp.step_a], R0s, M);
      for (int i = lane; i < A; i += 32) {
        const float4 d = __ldg(bt.atoms + a0 + i);
        const float3 u = apply_mt(M, T, d.x, d.y, d.z);
        S.u[i] = make_float4(u.x, u.y, u.z, d.w);
      }
      __syncwarp();

      // ---- optimize_pose: fragments in list order (P7-P10) ----
      int all_bumped = 0;
      for (int f = 0; f < F; ++f) {
        const uint4 fa = __ldg(bt.frags + 2 * (size_t)(f0 + f));
        const uint4 fb = __ldg(bt.frags + 2 * (size_t)(f0 + f) + 1);
        const unsigned mw[5] = {fa.x, fa.y, fa.z, fa.w, fb.x};
        const int ab = (int)(fb.y & 0xFFu), ae = (int)((fb.y >> 8) & 0xFFu);
        int nM = 0, nC = 0, base = 0;
#pragma unroll
        for (int s = 0; s < 5; ++s) {
          if (s * 32 >= A) break;
          const int i = s * 32 + lane;
          const bool in = i < A;
          const bool mv = in && ((mw[s] >> lane) & 1u);
          const bool cp = in && !mv && i != ab && i != ae;
          const unsigned bm = __ballot_sync(kFull, mv), bc = __ballot_sync(kFull, cp);
          if (mv) S.mlist[nM + __popc(bm & lt)] = (uint8_t)i;
          if (cp) S.wk[kMaxA - 1 - (nC + __popc(bc & lt))] = S.u[i];
          if (in && !mv) {
            const float4 p = S.u[i];
            base += grid_val(pk, node_index(g, p.x, p.y, p.z));
          }
          nM += __popc(bm);
          nC += __popc(bc);
        }
        base = warp_sum(base);
        const float4 pa = S.u[ab], pb = S.u[ae];
        const float3 a3 = make_float3(pa.x, pa.y, pa.z);
        float kx = 0.f, ky = 0.f, kz = 0.f;
        if (dp.n_t > 1) {
          const float vx = __fsub_rn(pb.x, pa.x), vy = __fsub_rn(pb.y, pa.y), vz = __fsub_rn(pb.z, pa.z);
          const float len = __fsqrt_rn(__fmaf_rn(vz, vz, __fmaf_rn(vy, vy, __fmul_rn(vx, vx))));
          if (!(len >= dp.eps_axis)) {  // DegenerateAxis
            degenerate = true;
            break;
          }
          kx = __fdiv_rn(vx, len);
          ky = __fdiv_rn(vy, len);
          kz = __fdiv_rn(vz, len);
        }
        // per-lane start of the lexicographic pair enumeration p = lane + 32*round
        const unsigned total = (unsigned)nM * (unsigned)nC;
        int pi = 0, pj = 0, qstep = 0, rstep = 0;
        if (nC > 0) {
          pi = lane / nC;
          pj = lane - pi * nC;
          qstep = 32 / nC;
          rstep = 32 - qstep * nC;
        }
        int best = INT_MIN, best_k = -1;
        for (int k = 0; k < dp.n_t; ++k) {
          float Rk[9];
          if (k > 0) {
            const float2 cs = pk.trig[k * dp.step_t];
            torsion_matrix(kx, ky, kz, cs.x, cs.y, Rk);
          }
          for (int m = lane; m < nM; m += 32) {
            const float4 p = S.u[S.mlist[m]];
            if (k == 0) {
              S.wk[m] = p;
            } else {
              const float3 q = torsion_apply(Rk, a3, p.x, p.y, p.z);
              S.wk[m] = make_float4(q.x, q.y, q.z, p.w);
            }
          }
          __syncwarp();
          // bump scan (P9): exists i in M, j in C' with d2 < bd2
          bool bumped = false;
          {
            int i = pi, j = pj;
            bool hit = false;
            for (unsigned b0 = 0; b0 < total; b0 += 32) {
              const unsigned p = b0 + (unsigned)lane;
              if (p < total) {
                const float4 x = S.wk[i];
                const float4 y = S.wk[kMaxA - 1 - j];
                hit |= dist2(x.x, x.y, x.z, y.x, y.y, y.z) < dp.bd2;
              }
              pairs_total += min(32u, total - b0);
              i += qstep;
              j += rstep;
              if (j >= nC) {
                j -= nC;
                ++i;
              }
              if (dp.early_exit && __any_sync(kFull, hit)) break;
            }
            bumped = __any_sync(kFull, hit);
          }
          ++evals;
          if (!bumped) {
            int sc = 0;
            for (int m = lane; m < nM; m += 32) {
              const float4 p = S.wk[m];
              sc += grid_val(pk, node_index(g, p.x, p.y, p.z));
            }
            sc = base + warp_sum(sc);
            if (sc > best) {
              best = sc;
              best_k = k;
            }
          } else if (dp.early_exit) {
            ++early_exits;
          }
          __syncwarp();
        }
        // commit the winner before the next fragment
        if (best_k > 0) {
          const float2 cs = pk.trig[best_k * dp.step_t];
          float Rk[9];
          torsion_matrix(kx, ky, kz, cs.x, cs.y, Rk);
          for (int m = lane; m < nM; m += 32) {
            const int i = S.mlist[m];
            const float4 p = S.u[i];
            const float3 q = torsion_apply(Rk, a3, p.x, p.y, p.z);
            S.u[i] = make_float4(q.x, q.y, q.z, p.w);
          }
        }
        if (best_k < 0) ++all_bumped;
        if (lane == 0) out.rtors[(size_t)(f0 + f) * dp.N + r] = best_k < 0 ? (uint8_t)DS_TORSION_NONE : (uint8_t)best_k;
        __syncwarp();
      }
      if (degenerate) break;
      // final geometric score + store the final pose
      int sc = 0;
      int hv = 0;
      for (int i = lane; i < A; i += 32) {
        const float4 p = S.u[i];
        sc += grid_val(pk, node_index(g, p.x, p.y, p.z));
        scr[(size_t)r * kMaxA + i] = p;
        hv += p.w != 0.f;
      }
      sc = warp_sum(sc);
      heavy = warp_sum(hv);
      const int valid = !(F >= 1 && all_bumped == F);  // P10
      if (lane == 0) {
        S.geom[r] = sc;
        S.valid[r] = valid;
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

    ds_result res;
    res.geom_score = 0;
    res.chem_fx = 0;
    res.best_restart = 0;
    res.best_ax = 0;
    res.best_ay = 0;
    res.n_kept = 0;
    res.poses_scored = (unsigned)(dp.N * dp.n_rot) + evals;
    res.bump_checks = pairs_total;
    res.bump_early_exits = early_exits;
    if (degenerate) {
      res.status = DS_STATUS_DEGENERATE_AXIS;
      if (lane == 0) out.res[lig] = res;
      __syncwarp();
      continue;
    }
    __syncwarp();
    // ---- select_poses (P12): order valid poses by (geom desc, restart asc) ----
    int nvalid = 0;
    for (int r = 0; r < dp.N; ++r) nvalid += S.valid[r];
    if (nvalid == 0) {
      res.status = DS_STATUS_NO_VALID_POSE;
      if (lane == 0) out.res[lig] = res;
      __syncwarp();
      continue;
    }
    for (int r = lane; r < dp.N; r += 32) {
      int rank = 0;
      if (S.valid[r]) {
        for (int q = 0; q < dp.N; ++q)
          rank += S.valid[q] && (S.geom[q] > S.geom[r] || (S.geom[q] == S.geom[r] && q < r));
        S.ord[rank] = r;
      }
      S.dis[r] = 0u;
    }
    __syncwarp();
    // pairwise dissimilarity of valid poses: heavy-atom sum of squared deltas in f64, atom order
    const int npairs = dp.N * (dp.N - 1) / 2;
    for (int pidx = lane; pidx < npairs; pidx += 32) {
      int p = 0, rem = pidx;
      while (rem >= dp.N - 1 - p) {
        rem -= dp.N - 1 - p;
        ++p;
      }
      const int q = p + 1 + rem;
      if (!S.valid[p] || !S.valid[q]) continue;
      double sum = 0.0;
      const float4 *up = scr + (size_t)p * kMaxA, *uq = scr + (size_t)q * kMaxA;
      for (int i = 0; i < A; ++i) {
        const float4 x = up[i], y = uq[i];
        if (x.w == 0.f) continue;
        const double dx = __dsub_rn((double)x.x, (double)y.x);
        const double dy = __dsub_rn((double)x.y, (double)y.y);
        const double dz = __dsub_rn((double)x.z, (double)y.z);
        double t = __dmul_rn(dx, dx);
        t = __dadd_rn(t, __dmul_rn(dy, dy));
        t = __dadd_rn(t, __dmul_rn(dz, dz));
        sum = __dadd_rn(sum, t);
      }
      if (heavy > 0 && sum >= __dmul_rn(dp.thr2, (double)heavy)) {
        atomicOr(&S.dis[p], 1u << q);
        atomicOr(&S.dis[q], 1u << p);
      }
    }
    __syncwarp();
    // greedy keep (warp-uniform)
    int kept[DS_MAX_RESTARTS];
    int nk = 0;
    for (int o = 0; o < nvalid && nk < dp.K; ++o) {
      const int c = S.ord[o];
      bool ok = true;
      for (int t = 0; t < nk; ++t) ok = ok && ((S.dis[c] >> kept[t]) & 1u);
      if (ok) kept[nk++] = c;
    }
    // ---- rescore kept poses (P11): exact fixed-point sum over (ligand atom, pocket atom) ----
    long long best_chem = 0;
    int best_r = -1;
    for (int t = 0; t < nk; ++t) {
      const int r = kept[t];
      long long acc = 0;
      const float4 *ur = scr + (size_t)r * kMaxA;
      for (int i = lane; i < A; i += 32) {
        const float4 x = ur[i];
        const int32_t *wrow = pk.wfx + (int)x.w * DS_N_TYPES * (pk.nb + 1);
        for (int j = 0; j < pk.n_atoms; ++j) {
          const float4 y = __ldg(pk.patoms + j);
          const float d2 = dist2(x.x, x.y, x.z, y.x, y.y, y.z);
          int b = 0;
#pragma unroll
          for (int q = 0; q < DS_MAX_BINS; ++q) b += (q < pk.nb) & !(d2 < pk.ub2[q]);
          acc += __ldg(wrow + (int)y.w * (pk.nb + 1) + b);
        }
      }
      acc = warp_sum64(acc);
      if (best_r < 0 || acc > best_chem || (acc == best_chem && r < best_r)) {
        best_chem = acc;
        best_r = r;
      }
      if (lane == 0 && out.rrec) out.rrec[(size_t)lig * dp.N + r].kept = (uint8_t)(t + 1);
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
    if (out.best_coords) {
      const float4 *ub = scr + (size_t)best_r * kMaxA;
      for (int i = lane; i < A; i += 32) {  // back to Å: q = fma(u, s, o)   (P2)
        const float4 x = ub[i];
        float *o = out.best_coords + 3 * (size_t)(a0 + i);
        o[0] = __fmaf_rn(x.x, pk.spacing, pk.ox);
        o[1] = __fmaf_rn(x.y, pk.spacing, pk.oy);
        o[2] = __fmaf_rn(x.z, pk.spacing, pk.oz);
      }
    }
    if (out.best_tors)
      for (int f = lane; f < F; f += 32) out.best_tors[f0 + f] = out.rtors[(size_t)(f0 + f) * dp.N + best_r];
    __syncwarp();
  }
}

size_t optimize_warp_smem_bytes() { return sizeof(OptWarpSmem); }

void launch_optimize_batched(const PocketView &pk, const BatchView &bt, const DockParams &dp, const int *order,
                             const uint32_t *keys, OptOut out, int *queue, int blocks, int warps, size_t smem,
                             cudaStream_t st) {
  cudaFuncSetAttribute(k_optimize_batched, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_optimize_batched<<<blocks, warps * 32, smem, st>>>(pk, bt, dp, order, keys, out, queue);
}

}  // namespace ds
