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

}  // namespace ds
