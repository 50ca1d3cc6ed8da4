// Per-op device entry points of the native slot (SPEC.md:183 grid_score, SPEC.md:203 rescore),
// batched over poses.  Input coordinates are in Å (pocket frame); they are mapped to the grid
// frame with the pinned u = fma(q, inv_s, -o/s) (DESIGN.md §3 P4).
#include "ds_kernels.cuh"

namespace ds {

__device__ __forceinline__ float to_grid(float q, float inv_s, float off) { return __fmaf_rn(q, inv_s, off); }

__global__ void k_grid_score(PocketView pk, const float *coords, int n_atoms, int n_poses, float offx, float offy,
                             float offz, int32_t *out) {
  const int pose = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (pose >= n_poses) return;
  int s = 0;
  for (int i = lane; i < n_atoms; i += 32) {
    const float *q = coords + 3 * ((size_t)pose * n_atoms + i);
    const int idx = node_index(pk.g, to_grid(q[0], pk.inv_s, offx), to_grid(q[1], pk.inv_s, offy),
                               to_grid(q[2], pk.inv_s, offz));
    s += (int)__ldg(pk.grid + idx) - 128;  // device grid is stored biased by +128
  }
  s = (int)__reduce_add_sync(kFull, (unsigned)s);
  if (lane == 0) out[pose] = s;
}

__global__ void k_rescore(PocketView pk, const float *coords, const uint8_t *types, int n_atoms, int n_poses,
                          float offx, float offy, float offz, int64_t *out) {
  __shared__ unsigned long long acc;
  const int pose = blockIdx.x;
  if (threadIdx.x == 0) acc = 0ull;
  __syncthreads();
  long long s = 0;
  for (int i = threadIdx.x; i < n_atoms; i += blockDim.x) {
    const float *q = coords + 3 * ((size_t)pose * n_atoms + i);
    const float ux = to_grid(q[0], pk.inv_s, offx), uy = to_grid(q[1], pk.inv_s, offy), uz = to_grid(q[2], pk.inv_s, offz);
    const int32_t *wrow = pk.wfx + (int)types[i] * DS_N_TYPES * (pk.nb + 1);
    for (int j = 0; j < pk.n_atoms; ++j) {
      const float4 y = __ldg(pk.patoms + j);
      const float d2 = dist2(ux, uy, uz, y.x, y.y, y.z);
      int b = 0;
#pragma unroll
      for (int k = 0; k < DS_MAX_BINS; ++k) b += (k < pk.nb) & !(d2 < pk.ub2[k]);
      s += __ldg(wrow + (int)y.w * (pk.nb + 1) + b);
    }
  }
  atomicAdd(&acc, (unsigned long long)s);
  __syncthreads();
  if (threadIdx.x == 0) out[pose] = (int64_t)acc;
}

static void offsets(const PocketView &pk, float *o) {
  o[0] = (float)(-(double)pk.ox / (double)pk.spacing);
  o[1] = (float)(-(double)pk.oy / (double)pk.spacing);
  o[2] = (float)(-(double)pk.oz / (double)pk.spacing);
}

void launch_grid_score(const PocketView &pk, const float *coords, int n_atoms, int n_poses, int32_t *out,
                       cudaStream_t st) {
  float o[3];
  offsets(pk, o);
  k_grid_score<<<(n_poses + 7) / 8, 256, 0, st>>>(pk, coords, n_atoms, n_poses, o[0], o[1], o[2], out);
}

void launch_rescore(const PocketView &pk, const float *coords, const uint8_t *types, int n_atoms, int n_poses,
                    float, int64_t *out, cudaStream_t st) {
  float o[3];
  offsets(pk, o);
  k_rescore<<<n_poses, 128, 0, st>>>(pk, coords, types, n_atoms, n_poses, o[0], o[1], o[2], out);
}

// ---- the other L2 ops of the slot in Å (SPEC.md:135 apply_rigid, :145 apply_torsion, :193
// bump_check), the pinned recipes of DESIGN.md §3 (P8, P9) evaluated in the Å frame; bit-identical
// to oracle/dock_oracle.c or_apply_rigid / or_apply_torsion / or_bump_check.

// thread per (pose, atom): w = p - c, p' = fma(m_i2, w_z, fma(m_i1, w_y, fma(m_i0, w_x, c_i)))
__global__ void k_apply_rigid(const float *coords, int n_atoms, int n_poses, const float *m, const float *center,
                              float *out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)n_atoms * n_poses) return;
  const int p = (int)(t / n_atoms);
  const float *M = m + 9 * p;
  const float3 c = make_float3(center[3 * p], center[3 * p + 1], center[3 * p + 2]);
  const float *q = coords + 3 * t;
  float R[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) R[k] = M[k];
  const float3 o = torsion_apply(R, c, q[0], q[1], q[2]);
  out[3 * t] = o.x;
  out[3 * t + 1] = o.y;
  out[3 * t + 2] = o.z;
}

// warp per pose: axis (every lane, same bits), DegenerateAxis (status 2, pose unchanged), lanes over atoms
__global__ void k_apply_torsion(const float *coords, int n_atoms, int n_poses, int ab, int ae, uint4 ma, unsigned mb,
                                float2 cs, int identity, float *out, int32_t *status) {
  const int pose = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (pose >= n_poses) return;
  const float *u = coords + 3 * (size_t)pose * n_atoms;
  float *o = out + 3 * (size_t)pose * n_atoms;
  const float3 a = make_float3(u[3 * ab], u[3 * ab + 1], u[3 * ab + 2]);
  const float vx = __fsub_rn(u[3 * ae], a.x), vy = __fsub_rn(u[3 * ae + 1], a.y), vz = __fsub_rn(u[3 * ae + 2], a.z);
  const float len = __fsqrt_rn(__fmaf_rn(vz, vz, __fmaf_rn(vy, vy, __fmul_rn(vx, vx))));
  const bool degen = !(len >= 1e-9f);
  float R[9];
  if (!degen && !identity)
    torsion_matrix(__fdiv_rn(vx, len), __fdiv_rn(vy, len), __fdiv_rn(vz, len), cs.x, cs.y, R);
  const unsigned w[5] = {ma.x, ma.y, ma.z, ma.w, mb};
  for (int i = lane; i < n_atoms; i += 32) {
    float3 q = make_float3(u[3 * i], u[3 * i + 1], u[3 * i + 2]);
    if (!degen && !identity && ((w[i >> 5] >> (i & 31)) & 1u)) q = torsion_apply(R, a, q.x, q.y, q.z);
    o[3 * i] = q.x;
    o[3 * i + 1] = q.y;
    o[3 * i + 2] = q.z;
  }
  if (lane == 0) status[pose] = degen ? 2 : 0;
}

// warp per pose: moving atoms i ascending (warp-uniform loop), lanes over the complement C' (not
// moving, not an axis atom) in 32-atom rounds; the sequential scan's pair count is the C' atoms of
// the rows before the first bump plus the rank of the first bumping j in its row, + 1 (P9, P14)
__global__ void k_bump_check(const float *coords, int n_atoms, int n_poses, int ab, int ae, uint4 ma, unsigned mb,
                             float bd2, int early_exit, uint8_t *bump, long long *pairs) {
  __shared__ uint8_t s_c[8][DS_MAX_ATOMS];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pose = blockIdx.x * (blockDim.x >> 5) + wib;
  if (pose >= n_poses) return;
  const float *u = coords + 3 * (size_t)pose * n_atoms;
  const unsigned w[5] = {ma.x, ma.y, ma.z, ma.w, mb};
  int nC = 0;
  for (int s = 0; s * 32 < n_atoms; ++s) {  // compaction of C'
    const int j = s * 32 + lane;
    const bool c = j < n_atoms && !((w[s] >> lane) & 1u) && j != ab && j != ae;
    const unsigned bc = __ballot_sync(kFull, c);
    if (c) s_c[wib][nC + __popc(bc & lanemask_lt())] = (uint8_t)j;
    nC += __popc(bc);
  }
  __syncwarp();
  long long n = 0;
  bool hit = false;
  for (int i = 0; i < n_atoms && !(hit && early_exit); ++i) {
    if (!((w[i >> 5] >> (i & 31)) & 1u)) continue;
    const float xi = u[3 * i], yi = u[3 * i + 1], zi = u[3 * i + 2];
    int first = -1;
    for (int c0 = 0; c0 < nC; c0 += 32) {
      bool b = false;
      if (c0 + lane < nC) {
        const int j = s_c[wib][c0 + lane];
        b = dist2(xi, yi, zi, u[3 * j], u[3 * j + 1], u[3 * j + 2]) < bd2;
      }
      const unsigned bb = __ballot_sync(kFull, b);
      if (bb && first < 0) first = c0 + __ffs(bb) - 1;
      if (bb && early_exit) break;
    }
    if (first >= 0) hit = true;
    n += (early_exit && first >= 0) ? first + 1 : nC;
  }
  if (lane == 0) {
    bump[pose] = hit ? 1 : 0;
    pairs[pose] = n;
  }
}

void launch_apply_rigid(const float *coords, int n_atoms, int n_poses, const float *m, const float *center, float *out,
                        cudaStream_t st) {
  const long long n = (long long)n_atoms * n_poses;
  k_apply_rigid<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(coords, n_atoms, n_poses, m, center, out);
}

void launch_apply_torsion(const float *coords, int n_atoms, int n_poses, int ab, int ae, const uint32_t *mask,
                          float2 cs, int identity, float *out, int32_t *status, cudaStream_t st) {
  k_apply_torsion<<<(n_poses + 7) / 8, 256, 0, st>>>(coords, n_atoms, n_poses, ab, ae,
                                                    make_uint4(mask[0], mask[1], mask[2], mask[3]), mask[4], cs,
                                                    identity, out, status);
}

void launch_bump_check(const float *coords, int n_atoms, int n_poses, int ab, int ae, const uint32_t *mask, float bd2,
                       int early_exit, uint8_t *bump, long long *pairs, cudaStream_t st) {
  k_bump_check<<<(n_poses + 7) / 8, 256, 0, st>>>(coords, n_atoms, n_poses, ab, ae,
                                                 make_uint4(mask[0], mask[1], mask[2], mask[3]), mask[4], bd2,
                                                 early_exit, bump, pairs);
}

// ---- build_pocket on the device (DESIGN.md §3 P18): thread per grid node, the
// pocket atoms staged in shared memory as f64; every operation is the host's (ds_host.cpp
// ds_build_pocket_grid) in the same order with explicit IEEE f64 rounding, so the grid is
// bit-identical to the host build.  37 M node-atom distances for the synthetic pocket.
__global__ void __launch_bounds__(256) k_build_pocket(const float *atom_xyz, int P, double ox, double oy, double oz,
                                                      double s, int nx, int ny, int nz, int32_t *values) {
  extern __shared__ double sa[];  // 3P
  for (int i = threadIdx.x; i < 3 * P; i += blockDim.x) sa[i] = (double)atom_xyz[i];
  __syncthreads();
  const long long n = (long long)nx * ny * nz;
  for (long long node = (long long)blockIdx.x * blockDim.x + threadIdx.x; node < n;
       node += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(node % nx), y = (int)((node / nx) % ny), z = (int)(node / ((long long)nx * ny));
    const double qx = __dadd_rn(ox, __dmul_rn((double)x, s));
    const double qy = __dadd_rn(oy, __dmul_rn((double)y, s));
    const double qz = __dadd_rn(oz, __dmul_rn((double)z, s));
    double best = __longlong_as_double(0x7FF0000000000000ll);
    for (int i = 0; i < P; ++i) {
      const double dx = __dsub_rn(qx, sa[3 * i]), dy = __dsub_rn(qy, sa[3 * i + 1]), dz = __dsub_rn(qz, sa[3 * i + 2]);
      const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      best = fmin(best, d2);
    }
    const double d = __dsqrt_rn(best);
    double g;
    if (d <= 3.0) g = __dadd_rn(-1.0, __ddiv_rn(__dmul_rn(2.0, d), 3.0));
    else if (d <= 5.0) g = 1.0;
    else if (d <= 8.0) g = __dsub_rn(1.0, __ddiv_rn(__dmul_rn(2.0, __dsub_rn(d, 5.0)), 3.0));
    else g = -1.0;
    values[node] = __double2int_rn(__dmul_rn(10.0, g));  // nearbyint: half-even
  }
}

void launch_build_pocket(const float *atom_xyz, int P, const double *origin, double s, const int *dims,
                         int32_t *values, int sm_count, cudaStream_t st) {
  const size_t smem = sizeof(double) * 3 * (size_t)P;
  allow_max_smem((const void *)k_build_pocket);
  k_build_pocket<<<sm_count * 8, 256, smem, st>>>(atom_xyz, P, origin[0], origin[1], origin[2], s, dims[0], dims[1],
                                                  dims[2], values);
}

}  // namespace ds
