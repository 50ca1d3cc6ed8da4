// Alignment (Alg. 1 lines 3-9) — batched family.
//
// One persistent CTA per SM stages the int8 pocket grid into shared memory once (the B200
// replacement for the paper's texture-cached pocket); each warp then pulls
// ligands from an atomic queue (LPT order) and scores all N x n_a^2 rigid poses of its ligand.
// Lanes own (restart, rotation) slots, R per lane, so every lane is busy for any atom count
// (the paper's lanes-over-atoms mapping idles lanes when A % 32 != 0); atoms are
// broadcast from a per-warp smem stage.  Output: one packed argmax key per (ligand, restart).
#include "ds_kernels.cuh"

namespace ds {

// dynamic smem layout: [grid bytes (16-aligned)] [trig_a float2[n_a]] [per warp: stage float4[32],
// params float[N*12], keys u32[N]]
__host__ __device__ inline int align_warp_smem_bytes(int N) { return 32 * 16 + ((N * 12 * 4 + N * 4 + 15) & ~15); }

template <int R, bool kSmemGrid>
__global__ void __launch_bounds__(1024, 1)
    k_align_batched(PocketView pk, BatchView bt, DockParams dp, const int *order, AlignOut out, int *queue) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gbytes = kSmemGrid ? pk.grid_bytes : 0;
  const int8_t *grid = pk.grid;
  if (kSmemGrid) {
    const int4 *src = reinterpret_cast<const int4 *>(pk.grid);
    int4 *dst = reinterpret_cast<int4 *>(smem);
    for (int i = threadIdx.x; i < gbytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    grid = reinterpret_cast<const int8_t *>(smem);
  }
  float2 *strig = reinterpret_cast<float2 *>(smem + gbytes);
  for (int i = threadIdx.x; i < dp.n_a; i += blockDim.x) strig[i] = pk.trig[i * dp.step_a];
  unsigned char *wbase = smem + gbytes + ((dp.n_a * 8 + 15) & ~15) + warp * align_warp_smem_bytes(dp.N);
  float4 *stage = reinterpret_cast<float4 *>(wbase);
  float *prm = reinterpret_cast<float *>(wbase + 32 * 16);
  unsigned *keys = reinterpret_cast<unsigned *>(prm + dp.N * 12);
  __syncthreads();

  const GridGeom g = pk.g;
  const int total = dp.N * dp.n_rot;
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(queue, 1);
    item = __shfl_sync(kFull, item, 0);
    if (item >= bt.L) break;
    const int lig = order ? order[item] : item;
    const int a0 = bt.atom_off[lig];
    const int A = bt.atom_off[lig + 1] - a0;
    const uint64_t idh = bt.idh[lig];
    for (int r = lane; r < dp.N; r += 32) {
      start_params(idh, dp.seed, r, pk.trig, pk.inv_s, g.nx, g.ny, g.nz, prm + r * 12, prm + r * 12 + 9);
      keys[r] = 0u;
    }
    const int nchunk = (A + 31) >> 5;
    if (nchunk == 1) stage[lane] = lane < A ? __ldg(bt.atoms + a0 + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();

    for (int base = 0; base < total; base += 32 * R) {
      float M[R][9], T[R][3];
      int score[R], rst[R], rot[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        int s = base + j * 32 + lane;
        s = s < total ? s : total - 1;
        const int r = s / dp.n_rot;
        const int q = s - r * dp.n_rot;
        const int ix = q / dp.n_a;
        const int iy = q - ix * dp.n_a;
        rst[j] = r;
        rot[j] = (base + j * 32 + lane) < total ? q : -1;
        const float *P = prm + r * 12;
        float R0s[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) R0s[k] = P[k];
        align_matrix(strig[ix], strig[iy], R0s, M[j]);
        T[j][0] = P[9];
        T[j][1] = P[10];
        T[j][2] = P[11];
        score[j] = 0;
      }
      for (int c = 0; c < nchunk; ++c) {
        if (nchunk > 1) {
          __syncwarp();
          const int ai = c * 32 + lane;
          stage[lane] = ai < A ? __ldg(bt.atoms + a0 + ai) : make_float4(0.f, 0.f, 0.f, 0.f);
          __syncwarp();
        }
        const int n = min(32, A - c * 32);
        for (int a = 0; a < n; ++a) {
          const float4 d = stage[a];
#pragma unroll
          for (int j = 0; j < R; ++j) {
            const float3 u = apply_mt(M[j], T[j], d.x, d.y, d.z);
            const int idx = node_index(g, u.x, u.y, u.z);
            score[j] += kSmemGrid ? (int)grid[idx] : (int)__ldg(grid + idx);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (rot[j] >= 0) atomicMax(&keys[rst[j]], ((unsigned)(score[j] + 32768) << 16) | (unsigned)(65535 - rot[j]));
    }
    __syncwarp();
    for (int r = lane; r < dp.N; r += 32) out.keys[(size_t)lig * dp.N + r] = keys[r];
    __syncwarp();
  }
}

int align_warp_smem_bytes_host(int N) { return align_warp_smem_bytes(N); }

void launch_align_batched(const PocketView &pk, const BatchView &bt, const DockParams &dp, const int *order,
                          AlignOut out, int *queue, int grid_in_smem, int blocks, int warps, size_t smem,
                          cudaStream_t st) {
  if (grid_in_smem) {
    cudaFuncSetAttribute(k_align_batched<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_align_batched<2, true><<<blocks, warps * 32, smem, st>>>(pk, bt, dp, order, out, queue);
  } else {
    cudaFuncSetAttribute(k_align_batched<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_align_batched<2, false><<<blocks, warps * 32, smem, st>>>(pk, bt, dp, order, out, queue);
  }
}

}  // namespace ds
