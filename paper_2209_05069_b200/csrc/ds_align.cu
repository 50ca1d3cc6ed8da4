// Alignment (Alg. 1 lines 3-9) — batched family.
//
// One persistent CTA per SM stages the int8 pocket grid (biased to uint8, with a one-node
// out-of-grid halo) into shared memory once — the B200 replacement for the paper's
// texture-cached pocket; each warp then pulls ligands from an atomic queue
// (LPT order) and scores all N x n_a^2 rigid poses of its ligand.
//
// Work split: a lane owns a (restart, ax) unit and sweeps every atom of the ligand for ALL ay.
// Because the pose is Ry(ay) (Rx(ax) (R0s d)) + t (DESIGN.md §3 P6), the inner vector
// v = Rx(ax) R0s d and the whole y coordinate (clamp and row offset included) are shared by the
// n_a values of ay.  For the default 12° step the 30 (cos, sin) pairs of ay are __constant__ and
// the ay loop is fully unrolled; angles are processed in pairs with Blackwell's packed f32x2
// FFMA2/FADD2 (each half bit-identical to the scalar __fmaf_rn/__fadd_rn of the recipe; the angle
// pairs become uniform-register operands), so per (atom, ay pair): 4 FFMA2 + 2 FADD2 + 4
// VIADDMNMX (unsigned clamp) + 4 IMAD + 2 LDS.U8 + 2 adds into scores packed two per register as
// biased 16-bit sums (9 SASS instructions per (atom, ay), 13.3 before f32x2).  The binding unit is
// the FMA-heavy pipe (FFMA2, FADD2 and IMAD all issue there; ncu: 82 % of its peak, shared-memory
// wavefronts 82 %), not issue.  Every lane is busy whatever the atom count (the paper's
// lanes-over-atoms mapping idles lanes when A % 32 != 0).  A round of the warp is
// one restart (lane = ax), so whether an atom's every pose of that restart stays within one node
// of the grid (|d| against the restart's translation, a bound with half a node of margin) is
// warp-uniform; such atoms (~70 % of the config-3 work) skip the two clamps and take both magic
// offsets out of the per-angle index: 262 instead of 322 SASS instructions per atom (-3.5 % align
// time measured: the shared-memory wavefronts of the random grid gathers bind next).  Output: one packed
// argmax key per (ligand, restart): (score + 32768) << 16 | (65535 - (ix * n_a + iy)).
#include <string.h>

#include <cooperative_groups.h>
#include <mutex>

#include "ds_kernels.cuh"

namespace ds {
namespace cg = cooperative_groups;

#ifndef DS_LAT_CS
#define DS_LAT_CS 8   // CTAs per (ligand, restart) cluster in the latency align kernel
#endif
#ifndef DS_LAT_W
#define DS_LAT_W 4    // warps per CTA there
#endif

__constant__ float4 c_trig_ay[360];  // (cos, sin, -sin, 0) of iy * step_a
// the same angles as packed pairs for the f32x2 path: [k/2] = {(c_k, c_k+1), (s_k, s_k+1), (-s_k, -s_k+1)}
__constant__ unsigned long long c_pair_ay[180][3];

#ifndef DS_ALIGN_INSIDE
#define DS_ALIGN_INSIDE 1  // unclamped node indices for atoms whose poses all stay in the grid
#endif
#ifndef DS_ALIGN_F32X2
#define DS_ALIGN_F32X2 2   // 0 scalar, 1 all packed, 2 packed x + scalar z (fastest), 3 packed FMAs + scalar rounding adds
#endif

// dynamic smem layout: [grid bytes (16-aligned)] [trig_a float4[n_a]] [per warp: stage float4[32],
// params float[N*kPrm], keys u32[N]]
// params per restart: R0s (9), t (3), the unclamped-path radius limit (1)
constexpr int kPrm = 13;
__host__ __device__ inline int align_warp_smem_bytes(int N) { return 32 * 16 + ((N * kPrm * 4 + N * 4 + 15) & ~15); }

__device__ __forceinline__ unsigned grid_u8(const uint8_t *grid, int idx, bool smem) {
  return smem ? (unsigned)grid[idx] : (unsigned)__ldg(grid + idx);
}

// f32x2 form of unit_atom for the constant-angle path: per pair of angles (k, k+1)
//   UX = fma2(S, VZ, fma2(C, VX, TX)),  UZ = fma2(C, VZ, fma2(-S, VX, TZ)),  + (magic, magic)
// — lane-for-lane the same operations as the scalar recipe P6/P4, in half the FP32 issue slots.
template <int G, bool kSmemGrid>
__device__ __forceinline__ void unit_atom_x2(const float3 v, f2_t TX, f2_t TZ, unsigned yk, const GridGeom &g,
                                             const uint8_t *grid, unsigned *acc) {
  const f2_t VX = f2_pack(v.x, v.x), VZ = f2_pack(v.z, v.z);
  const f2_t MM = f2_pack(kMagic, kMagic);
#pragma unroll
  for (int k = 0; k < G; k += 2) {
    const f2_t C = c_pair_ay[k >> 1][0], S = c_pair_ay[k >> 1][1], NS = c_pair_ay[k >> 1][2];
#if DS_ALIGN_F32X2 == 3  // packed FMAs, scalar magic adds (FADD may issue on the FMA-lite pipe)
    float ux0, ux1, uz0, uz1;
    f2_unpack(f2_fma(S, VZ, f2_fma(C, VX, TX)), ux0, ux1);
    f2_unpack(f2_fma(C, VZ, f2_fma(NS, VX, TZ)), uz0, uz1);
    const float mx0 = __fadd_rn(ux0, kMagic), mx1 = __fadd_rn(ux1, kMagic);
    const float mz0 = __fadd_rn(uz0, kMagic), mz1 = __fadd_rn(uz1, kMagic);
#elif DS_ALIGN_F32X2 == 2  // packed x, scalar z
    float mx0, mx1;
    f2_unpack(f2_add(f2_fma(S, VZ, f2_fma(C, VX, TX)), MM), mx0, mx1);
    float c0, c1, s0, s1;
    f2_unpack(C, c0, c1);
    f2_unpack(S, s0, s1);
    float vx, vz, tz, tz1;
    f2_unpack(VX, vx, tz1);
    f2_unpack(VZ, vz, tz1);
    f2_unpack(TZ, tz, tz1);
    const float mz0 = __fadd_rn(__fmaf_rn(c0, vz, __fmaf_rn(-s0, vx, tz)), kMagic);
    const float mz1 = __fadd_rn(__fmaf_rn(c1, vz, __fmaf_rn(-s1, vx, tz)), kMagic);
#else
    const f2_t UX = f2_add(f2_fma(S, VZ, f2_fma(C, VX, TX)), MM);
    const f2_t UZ = f2_add(f2_fma(C, VZ, f2_fma(NS, VX, TZ)), MM);
    float mx0, mx1, mz0, mz1;
    f2_unpack(UX, mx0, mx1);
    f2_unpack(UZ, mz0, mz1);
#endif
    const unsigned K = (unsigned)(kMagicBits - 1);
    const unsigned cx0 = min((unsigned)__float_as_int(mx0) - K, (unsigned)(g.nx + 1));
    const unsigned cx1 = min((unsigned)__float_as_int(mx1) - K, (unsigned)(g.nx + 1));
    const unsigned cz0 = min((unsigned)__float_as_int(mz0) - K, (unsigned)(g.nz + 1));
    const unsigned cz1 = min((unsigned)__float_as_int(mz1) - K, (unsigned)(g.nz + 1));
    const int i0 = (int)((cx0 + g.NXY * cz0) + yk);
    const int i1 = (int)((cx1 + g.NXY * cz1) + yk);
    acc[k >> 1] += grid_u8(grid, i0, kSmemGrid) + (grid_u8(grid, i1, kSmemGrid) << 16);
  }
}

// The same scores for an atom whose every alignment pose stays within one node of the grid (the
// caller's radius test): no clamp can bind, so the node index is bits(mx) + NXY bits(mz) + ykf with
// both magic offsets folded into the per-atom ykf — one IADD + one IMAD per angle instead of two
// unsigned clamps + IMAD + IADD; identical indices (the clamps are identities here).
template <int G, bool kSmemGrid>
__device__ __forceinline__ void unit_atom_x2_inside(const float3 v, f2_t TX, f2_t TZ, unsigned ykf, const GridGeom &g,
                                                    const uint8_t *grid, unsigned *acc) {
  const f2_t VX = f2_pack(v.x, v.x), VZ = f2_pack(v.z, v.z);
  const f2_t MM = f2_pack(kMagic, kMagic);
#pragma unroll
  for (int k = 0; k < G; k += 2) {
    const f2_t C = c_pair_ay[k >> 1][0], S = c_pair_ay[k >> 1][1];
    float mx0, mx1;
    f2_unpack(f2_add(f2_fma(S, VZ, f2_fma(C, VX, TX)), MM), mx0, mx1);
    float c0, c1, s0, s1;
    f2_unpack(C, c0, c1);
    f2_unpack(S, s0, s1);
    float vx, vz, tz, tz1;
    f2_unpack(VX, vx, tz1);
    f2_unpack(VZ, vz, tz1);
    f2_unpack(TZ, tz, tz1);
    const float mz0 = __fadd_rn(__fmaf_rn(c0, vz, __fmaf_rn(-s0, vx, tz)), kMagic);
    const float mz1 = __fadd_rn(__fmaf_rn(c1, vz, __fmaf_rn(-s1, vx, tz)), kMagic);
    const int i0 = (int)(g.NXY * (unsigned)__float_as_int(mz0) + ((unsigned)__float_as_int(mx0) + ykf));
    const int i1 = (int)(g.NXY * (unsigned)__float_as_int(mz1) + ((unsigned)__float_as_int(mx1) + ykf));
    acc[k >> 1] += grid_u8(grid, i0, kSmemGrid) + (grid_u8(grid, i1, kSmemGrid) << 16);
  }
}

// Accumulate the biased grid values of angles iy = iy0 .. iy0+G-1 for one atom's v into G/2
// packed registers (low half: even k, high half: odd k).
template <int G, bool kConst, bool kSmemGrid>
__device__ __forceinline__ void unit_atom(const float3 v, const float *t, unsigned yk, const GridGeom &g,
                                          const uint8_t *grid, const float4 *strig, int iy0, int n_a,
                                          unsigned *acc) {
#if DS_ALIGN_F32X2
  if (kConst) {
    unit_atom_x2<G, kSmemGrid>(v, f2_pack(t[0], t[0]), f2_pack(t[2], t[2]), yk, g, grid, acc);
    return;
  }
#endif
#pragma unroll
  for (int k = 0; k < G; k += 2) {
    const float4 c0 = kConst ? c_trig_ay[k] : strig[min(iy0 + k, n_a - 1)];
    const float4 c1 = kConst ? c_trig_ay[k + 1] : strig[min(iy0 + k + 1, n_a - 1)];
    const float ux0 = __fmaf_rn(c0.y, v.z, __fmaf_rn(c0.x, v.x, t[0]));
    const float uz0 = __fmaf_rn(c0.x, v.z, __fmaf_rn(c0.z, v.x, t[2]));
    const float ux1 = __fmaf_rn(c1.y, v.z, __fmaf_rn(c1.x, v.x, t[0]));
    const float uz1 = __fmaf_rn(c1.x, v.z, __fmaf_rn(c1.z, v.x, t[2]));
    const int i0 = (int)(clamp_bits(ux0, g.nx + 1) + g.NXY * clamp_bits(uz0, g.nz + 1) + yk);
    const int i1 = (int)(clamp_bits(ux1, g.nx + 1) + g.NXY * clamp_bits(uz1, g.nz + 1) + yk);
    acc[k >> 1] += grid_u8(grid, i0, kSmemGrid) + (grid_u8(grid, i1, kSmemGrid) << 16);
  }
}

// NA > 0: n_a == NA fixed (G == NA, one unit per (restart, ax)); NA == 0: runtime n_a, ay in chunks
// of G with units ordered chunk-major so a warp round shares its chunk.
template <int NA, int G, bool kSmemGrid>
#ifndef DS_ALIGN_WARPS
#define DS_ALIGN_WARPS 32
#endif
__global__ void __launch_bounds__(DS_ALIGN_WARPS * 32, 1)
    k_align_batched(PocketView pk, BatchView bt, DockParams dp, const int *order, AlignOut out, int *queue) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr bool kConst = NA > 0;
  static_assert(G % 2 == 0, "scores are packed in pairs");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_a = kConst ? NA : dp.n_a;
  const int gbytes = kSmemGrid ? pk.grid_bytes : 0;
  const uint8_t *grid = pk.grid;
  if (kSmemGrid) {
    const int4 *src = reinterpret_cast<const int4 *>(pk.grid);
    int4 *dst = reinterpret_cast<int4 *>(smem);
    for (int i = threadIdx.x; i < gbytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    grid = smem;
  }
  float4 *strig = reinterpret_cast<float4 *>(smem + gbytes);
  for (int i = threadIdx.x; i < n_a; i += blockDim.x) {
    const float2 cs = pk.trig[i * dp.step_a];
    strig[i] = make_float4(cs.x, cs.y, -cs.y, 0.f);
  }
  unsigned char *wbase = smem + gbytes + n_a * 16 + warp * align_warp_smem_bytes(dp.N);
  float4 *stage = reinterpret_cast<float4 *>(wbase);
  float *prm = reinterpret_cast<float *>(wbase + 32 * 16);
  unsigned *keys = reinterpret_cast<unsigned *>(prm + dp.N * kPrm);
  __syncthreads();

  const GridGeom g = pk.g;
  const int nch = kConst ? 1 : (n_a + G - 1) / G;   // ay chunks
  const int per_h = dp.N * n_a;                        // units per chunk: (restart, ax)
  const int total = nch * per_h;
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
      float *P = prm + r * kPrm;
      start_params(idh, dp.seed, r, pk.trig, pk.inv_s, g.nx, g.ny, g.nz, P, P + 9);
      // unclamped path (kConst): an atom with |d|^2 < P[12] has every pose of this restart within
      // one node of the grid in x and z — |u - t| <= |v| (1 + 1e-5) + 1e-5 and |v| <= |d| inv_s
      // (1 + 1e-5), so |d| inv_s <= rs = min(t + 1, n - t) with the 0.9996 factor keeps u in
      // [-1.5, n + 0.5], i.e. rint(u) + 1 in [0, n + 1] (the halo planes included)
      const float rs = fminf(fminf(__fadd_rn(P[9], 1.f), __fsub_rn((float)g.nx, P[9])),
                             fminf(__fadd_rn(P[11], 1.f), __fsub_rn((float)g.nz, P[11])));
      const float ra = __fmul_rn(rs, pk.spacing);  // spacing * inv_s = 1 within 2^-23
      P[12] = __fmul_rn(__fmul_rn(ra, ra), 0.9996f);
      keys[r] = 0u;
    }
    const int nchunk = (A + 31) >> 5;
    // staged atoms carry |d|^2 in .w (the alignment does not read the type)
    auto stage_atom = [&](int ai) {
      if (ai >= A) return make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 d = __ldg(bt.atoms + a0 + ai);
      return make_float4(d.x, d.y, d.z, __fmaf_rn(d.z, d.z, __fmaf_rn(d.y, d.y, __fmul_rn(d.x, d.x))));
    };
    if (nchunk == 1) stage[lane] = stage_atom(lane);
    __syncwarp();

    // kConst: one restart per round (units padded to 32 per restart, unit = 32 r + ax), so the
    // restart's parameters and the unclamped-path test are warp-uniform; else 32 (chunk, restart,
    // ax) units per round.  (The opaque XOR hides that r is warp-uniform: uniform r moves the
    // restart's values into uniform registers and evicts the ay constants from them.)
    const int total_u = kConst ? dp.N * 32 : total;
    for (int base = 0; base < total_u; base += 32) {
      const int unit = kConst ? base + (lane ^ (int)dp.opaque0) : min(base + lane, total - 1);
      const bool uvalid = kConst ? (unit & 31) < n_a : base + lane < total;
      const int h = kConst ? 0 : unit / per_h;
      const int q = unit - h * per_h;
      const int r = kConst ? unit >> 5 : q / n_a;
      const int ix = kConst ? min(unit & 31, n_a - 1) : q - r * n_a;
      const int iy0 = h * G;
      const float *P = prm + r * kPrm;
      float Rp[9], t[3];
      {
        float R0s[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) R0s[k] = P[k];
        const float4 cx = strig[ix];
        align_rx(make_float2(cx.x, cx.y), R0s, Rp);
        t[0] = P[9];
        t[1] = P[10];
        t[2] = P[11];
      }
      const float lim = P[12];  // the unclamped path's |d|^2 limit of this round's restart
      unsigned acc[G / 2];
#pragma unroll
      for (int k = 0; k < G / 2; ++k) acc[k] = 0u;
      for (int c = 0; c < nchunk; ++c) {
        if (nchunk > 1) {
          __syncwarp();
          stage[lane] = stage_atom(c * 32 + lane);
          __syncwarp();
        }
        const int n = min(32, A - c * 32);
        for (int a = 0; a < n; ++a) {
          const float4 d = stage[a];
          const float3 v = align_v(Rp, d.x, d.y, d.z);
          // u_y is shared by all ay; the opaque XOR keeps the row offset an ALU add per angle
          const unsigned yk = (g.NX * clamp_bits(__fadd_rn(v.y, t[1]), g.ny + 1)) ^ dp.opaque0;
#if DS_ALIGN_F32X2 == 2 && DS_ALIGN_INSIDE
          if (kConst && d.w < lim) {  // the restart keeps every pose of the atom inside (warp-uniform)
            const unsigned K = (unsigned)(kMagicBits - 1);
            // opaque: no constant folded out of ykf into the shared-memory address (it would need the
            // window base in a vector register and an extra add per load)
            unit_atom_x2_inside<G, kSmemGrid>(v, f2_pack(t[0], t[0]), f2_pack(t[2], t[2]),
                                              (yk - K - g.NXY * K) ^ dp.opaque0, g, grid, acc);
            continue;
          }
#endif
          unit_atom<G, kConst, kSmemGrid>(v, t, yk, g, grid, strig, iy0, n_a, acc);
        }
      }
      unsigned best = 0u;
      const int bias = 128 * A;  // the device grid stores v + 128
#pragma unroll
      for (int k = 0; k < G; ++k) {
        const int iy = iy0 + k;
        const int sc = (int)((acc[k >> 1] >> (16 * (k & 1))) & 0xFFFFu) - bias;
        if (iy < n_a) best = max(best, ((unsigned)(sc + 32768) << 16) | (unsigned)(65535 - (ix * n_a + iy)));
      }
      if (uvalid) atomicMax(&keys[r], best);
    }
    __syncwarp();
    for (int r = lane; r < dp.N; r += 32) out.keys[(size_t)lig * dp.N + r] = keys[r];
    __syncwarp();
  }
}

// ---- latency family: one ligand spread over the GPU -----------------------
// Block (ligand, restart, atom chunk) = one warp; lane = ax.  Each lane scores its ax for every ay
// over the chunk's atoms (grid read through L1 from the biased global copy) and adds the partial
// sums into scores[(lig*N + r) * n_rot + ax*n_a + ay] with global atomics; the optimisation
// kernel takes the argmax.  ACH atoms per block keeps ~A/ACH x N blocks in flight.
template <int NA>
__global__ void __launch_bounds__(32)
    k_align_latency(PocketView pk, BatchView bt, DockParams dp, int ach, int nchunks, int *scores) {
  constexpr bool kConst = NA > 0;
  constexpr int G = kConst ? NA : 8;
  const int lane = threadIdx.x;
  const int lig = blockIdx.x / (dp.N * nchunks);
  const int rem = blockIdx.x - lig * dp.N * nchunks;
  const int r = rem / nchunks;
  const int c = rem - r * nchunks;
  const int a0 = bt.atom_off[lig];
  const int A = bt.atom_off[lig + 1] - a0;
  const int c0 = c * ach, c1 = min(A, c0 + ach);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (c0 >= A) return;
  __shared__ float4 strig[360];
  const int n_a = kConst ? NA : dp.n_a;
  for (int i = lane; i < n_a; i += 32) {
    const float2 cs = pk.trig[i * dp.step_a];
    strig[i] = make_float4(cs.x, cs.y, -cs.y, 0.f);
  }
  __syncwarp();
  const GridGeom g = pk.g;
  float R0s[9], t[3];
  start_params(bt.idh[lig], dp.seed, r, pk.trig, pk.inv_s, g.nx, g.ny, g.nz, R0s, t);
  int *sc = scores + ((size_t)lig * dp.N + r) * dp.n_rot;
  for (int ix = lane; ix < n_a; ix += 32) {
    float Rp[9];
    const float4 cx = strig[ix];
    align_rx(make_float2(cx.x, cx.y), R0s, Rp);
    for (int iy0 = 0; iy0 < n_a; iy0 += G) {
      unsigned acc[G / 2];
#pragma unroll
      for (int k = 0; k < G / 2; ++k) acc[k] = 0u;
      for (int a = c0; a < c1; ++a) {
        const float4 d = __ldg(bt.atoms + a0 + a);
        const float3 v = align_v(Rp, d.x, d.y, d.z);
        const unsigned yk = g.NX * clamp_bits(__fadd_rn(v.y, t[1]), g.ny + 1);
        unit_atom<G, kConst, false>(v, t, yk, g, pk.grid, strig, iy0, n_a, acc);
      }
      const int bias = 128 * (c1 - c0);
#pragma unroll
      for (int k = 0; k < G; ++k)
        if (iy0 + k < n_a) atomicAdd(sc + ix * n_a + iy0 + k, (int)((acc[k >> 1] >> (16 * (k & 1))) & 0xFFFFu) - bias);
    }
  }
}

// the n_a = 30 angle table in __constant__ (scalar and packed-pair forms); same values as the ctx
// trig table (P0), identical for every caller (n_a = 30 <=> step_a = 12), so it is uploaded once
// per device (a blocking copy, so no stream can launch before it lands) instead of per call
static void upload_const_angles(int step_a, cudaStream_t) {
  static std::mutex mu;
  static bool done[256];
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (dev >= 0 && dev < 256 && done[dev]) return;
  float4 h[30];
  unsigned long long hp[15][3];
  for (int i = 0; i < 30; ++i) {
    const double rad = (double)(i * step_a) * 0.017453292519943295;
    const float c = (float)cos(rad), s = (float)sin(rad);
    h[i] = make_float4(c, s, -s, 0.f);
  }
  auto pk = [](float lo, float hi) {
    unsigned a, b;
    memcpy(&a, &lo, 4);
    memcpy(&b, &hi, 4);
    return (unsigned long long)a | ((unsigned long long)b << 32);
  };
  for (int p = 0; p < 15; ++p) {
    hp[p][0] = pk(h[2 * p].x, h[2 * p + 1].x);
    hp[p][1] = pk(h[2 * p].y, h[2 * p + 1].y);
    hp[p][2] = pk(h[2 * p].z, h[2 * p + 1].z);
  }
  if (cudaMemcpyToSymbol(c_trig_ay, h, sizeof h) == cudaSuccess &&
      cudaMemcpyToSymbol(c_pair_ay, hp, sizeof hp) == cudaSuccess && dev >= 0 && dev < 256)
    done[dev] = true;
}

// ---- latency family, n_a = 30: one thread-block cluster per (ligand, restart) ---------------
// CS CTAs x W warps split the ligand's atoms into CS*W contiguous ranges; lane = ax scores every
// ay over its warp's range (packed f32x2 path, grid through L1).  The 900 partial sums are added
// across the CTA's warps in shared memory, then across the cluster through distributed shared
// memory (CTA k sums rotation slice k over all CS CTAs and folds its best key into CTA 0 with a
// DSMEM atomicMax) — no global atomics, no scores buffer to clear, and the optimisation kernel
// reads one key per (ligand, restart).  Integer sums: the key is exactly the argmax of the
// single-pass sum (ties -> smallest rotation index).
template <int CS, int W>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(W * 32)
    k_align_latency_cl(PocketView pk, BatchView bt, DockParams dp, unsigned *keys) {
  constexpr int NA = 30, NR = NA * NA, SL = (NR + CS - 1) / CS;
  // the optimisation kernel may launch now (programmatic dependent launch): it stages its shared
  // memory while this kernel runs and waits (griddepcontrol.wait) before reading the keys
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ int part[W][NR];
  __shared__ unsigned s_best;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = blockIdx.x / CS;
  const int lig = lr / dp.N, r = lr - lig * dp.N;
  const int a0 = bt.atom_off[lig], A = bt.atom_off[lig + 1] - a0;
  const int gw = rank * W + warp;
  const int c0 = A * gw / (CS * W), c1 = A * (gw + 1) / (CS * W);
  if (threadIdx.x == 0) s_best = 0u;
  const GridGeom g = pk.g;
  float R0s[9], t[3];
  start_params(bt.idh[lig], dp.seed, r, pk.trig, pk.inv_s, g.nx, g.ny, g.nz, R0s, t);
  if (lane < NA) {
    float Rp[9];
    align_rx(pk.trig[lane * dp.step_a], R0s, Rp);
    unsigned acc[NA / 2];
#pragma unroll
    for (int k = 0; k < NA / 2; ++k) acc[k] = 0u;
    for (int a = c0; a < c1; ++a) {
      const float4 d = __ldg(bt.atoms + a0 + a);
      const float3 v = align_v(Rp, d.x, d.y, d.z);
      const unsigned yk = g.NX * clamp_bits(__fadd_rn(v.y, t[1]), g.ny + 1);
      unit_atom<NA, true, false>(v, t, yk, g, pk.grid, nullptr, 0, NA, acc);
    }
    const int bias = 128 * (c1 - c0);
#pragma unroll
    for (int k = 0; k < NA; ++k) part[warp][lane * NA + k] = (int)((acc[k >> 1] >> (16 * (k & 1))) & 0xFFFFu) - bias;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < NR; q += W * 32) {
    int s = part[0][q];
#pragma unroll
    for (int w = 1; w < W; ++w) s += part[w][q];
    part[0][q] = s;
  }
  cl.sync();
  unsigned best = 0u;
  for (int q = rank * SL + (int)threadIdx.x; q < min(NR, (rank + 1) * SL); q += W * 32) {
    int s = 0;
#pragma unroll
    for (int k = 0; k < CS; ++k) s += cl.map_shared_rank(&part[0][0], k)[q];
    best = max(best, ((unsigned)(s + 32768) << 16) | (unsigned)(65535 - q));
  }
  best = __reduce_max_sync(kFull, best);
  if (lane == 0 && best) atomicMax(cl.map_shared_rank(&s_best, 0), best);
  cl.sync();  // also keeps every CTA's shared memory alive until all remote reads are done
  if (rank == 0 && threadIdx.x == 0) keys[lr] = s_best;
}

// returns true when the cluster kernel wrote one key per (ligand, restart) into keys (n_a = 30),
// false when the generic kernel accumulated into scores
bool launch_align_latency(const PocketView &pk, const BatchView &bt, const DockParams &dp, int max_atoms, int *scores,
                          unsigned *keys, cudaStream_t st) {
  if (dp.n_a == 30) {
    upload_const_angles(dp.step_a, st);
    k_align_latency_cl<DS_LAT_CS, DS_LAT_W><<<bt.L * dp.N * DS_LAT_CS, DS_LAT_W * 32, 0, st>>>(pk, bt, dp, keys);
    return true;
  }
  const int ach = 4;
  const int nchunks = (max_atoms + ach - 1) / ach;
  const int blocks = bt.L * dp.N * nchunks;
  k_align_latency<0><<<blocks, 32, 0, st>>>(pk, bt, dp, ach, nchunks, scores);
  return false;
}

int align_warp_smem_bytes_host(int N) { return align_warp_smem_bytes(N); }

template <int NA, int G, bool S>
static void launch_t(const PocketView &pk, const BatchView &bt, const DockParams &dp, const int *order, AlignOut out,
                     int *queue, int blocks, int warps, size_t smem, cudaStream_t st) {
  allow_max_smem((const void *)k_align_batched<NA, G, S>);
  k_align_batched<NA, G, S><<<blocks, warps * 32, smem, st>>>(pk, bt, dp, order, out, queue);
}

// resident CTAs per SM of the default-step alignment kernel (grid in shared memory) for this
// launch shape: the occupancy API on the real kernel (ds_query_capacity)
int align_blocks_per_sm(int warps, size_t smem) {
  int n = 0;
  allow_max_smem((const void *)k_align_batched<30, 30, true>);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_align_batched<30, 30, true>, warps * 32, smem);
  return n;
}

void launch_align_batched(const PocketView &pk, const BatchView &bt, const DockParams &dp, const int *order,
                          AlignOut out, int *queue, int grid_in_smem, int blocks, int warps, size_t smem,
                          cudaStream_t st) {
  if (dp.n_a == 30) {  // default 12° step: all 30 ay per unit, constant-bank angles
    upload_const_angles(dp.step_a, st);
    if (grid_in_smem) launch_t<30, 30, true>(pk, bt, dp, order, out, queue, blocks, warps, smem, st);
    else launch_t<30, 30, false>(pk, bt, dp, order, out, queue, blocks, warps, smem, st);
  } else {
    if (grid_in_smem) launch_t<0, 8, true>(pk, bt, dp, order, out, queue, blocks, warps, smem, st);
    else launch_t<0, 8, false>(pk, bt, dp, order, out, queue, blocks, warps, smem, st);
  }
}

}  // namespace ds
