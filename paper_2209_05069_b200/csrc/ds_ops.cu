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
  cudaFuncSetAttribute(k_build_pocket, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_build_pocket<<<sm_count * 8, 256, smem, st>>>(atom_xyz, P, origin[0], origin[1], origin[2], s, dims[0], dims[1],
                                                  dims[2], values);
}

}  // namespace ds
