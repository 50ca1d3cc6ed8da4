// Device-side numeric primitives of the docking hot path (sm_100a).
//
// Every function here implements one pin of the numeric recipe and must stay
// bit-identical to the CPU restatement in oracle/.  The translation unit is compiled with
// --fmad=false, so a*b+c is two roundings unless written as __fmaf_rn / fma explicitly.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dockscreen.h"

namespace ds {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr float kMagic = 12582912.0f;     // 1.5 * 2^23: x + kMagic rounds x half-even to an integer
constexpr int kMagicBits = 0x4B400000;    // bit pattern of kMagic
constexpr int kOutside = -100;            // out-of-grid penalty per atom
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr int kChemShift = 24;            // chem fixed point 2^-24 (P11)

// ---- P5: counter-based starting-pose PRNG (SplitMix64 finaliser) --------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ---- P1: pinned f32 3x3 product C = A (x) B, C_ij = fma(A_i2,B_2j, fma(A_i1,B_1j, A_i0*B_0j))
__device__ __forceinline__ void matmul3(const float *A, const float *B, float *C) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      C[3 * i + j] = __fmaf_rn(A[3 * i + 2], B[6 + j], __fmaf_rn(A[3 * i + 1], B[3 + j], __fmul_rn(A[3 * i], B[j])));
}

// ---- P3: pose transform u = M d + t, u_k = fma(M_k2,d.z, fma(M_k1,d.y, fma(M_k0,d.x,t_k)))
__device__ __forceinline__ float3 apply_mt(const float *M, const float *t, float dx, float dy, float dz) {
  float3 u;
  u.x = __fmaf_rn(M[2], dz, __fmaf_rn(M[1], dy, __fmaf_rn(M[0], dx, t[0])));
  u.y = __fmaf_rn(M[5], dz, __fmaf_rn(M[4], dy, __fmaf_rn(M[3], dx, t[1])));
  u.z = __fmaf_rn(M[8], dz, __fmaf_rn(M[7], dy, __fmaf_rn(M[6], dx, t[2])));
  return u;
}

// ---- P4: nearest node (round half-even) + in-grid test, as an index into the PADDED grid.
// The device grid carries a one-node halo holding kOutside on every side, so the in-grid test is
// one unsigned clamp per axis: c = min(bits(u + 1.5*2^23) - (kMagicBits - 1), n + 1) is rint(u) + 1
// for in-range nodes and lands in a halo plane (0 or n + 1) otherwise — below-range values wrap
// to huge unsigned and clamp to n + 1 (VIADDMNMX: one instruction).  For |u| < 2^22 the magic add
// equals rintf; every |u| >= 2^22, inf or NaN lands in the halo (dims < 2^21), exactly like the
// oracle's float test 0 <= rint(u) <= n-1.
struct GridGeom {
  int nx, ny, nz;          // interior dims
  unsigned NX, NXY;        // padded row / plane pitch: nx+2, (nx+2)(ny+2)
  unsigned bx, by, bz;     // nx+1, ny+1, nz+1: index of the far halo plane (the clamp bound)
};
// bound = n + 1
__device__ __forceinline__ unsigned clamp_bits(float u, unsigned bound) {
  const unsigned b = (unsigned)__float_as_int(__fadd_rn(u, kMagic)) - (unsigned)(kMagicBits - 1);
  return min(b, bound);
}
// node index from coordinates that already carry the +1.5*2^23 magic add (packed callers)
__device__ __forceinline__ int node_index_magic(const GridGeom &g, float mx, float my, float mz) {
  const unsigned K = (unsigned)(kMagicBits - 1);
  return (int)(min((unsigned)__float_as_int(mx) - K, g.bx) + g.NX * min((unsigned)__float_as_int(my) - K, g.by) +
               g.NXY * min((unsigned)__float_as_int(mz) - K, g.bz));
}
__device__ __forceinline__ int node_index(const GridGeom &g, float ux, float uy, float uz) {
  return (int)(clamp_bits(ux, g.bx) + g.NX * clamp_bits(uy, g.by) + g.NXY * clamp_bits(uz, g.bz));
}

// ---- P5: starting pose parameters of restart r: R0s = (Rz(g) (x) (Ry(b) (x) Rx(a))) * inv_s,
// t = (n-1) * (0.1 + 0.8 U)   (grid frame)
__device__ __forceinline__ void start_params(uint64_t idh, int64_t seed, int r, const float2 *trig, float inv_s,
                                             int nx, int ny, int nz, float *R0s, float *t) {
  const uint64_t base = idh ^ ((uint64_t)seed * kGolden);
  uint64_t z[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) z[k] = mix64(base + (uint64_t)(r * 8 + k + 1) * kGolden);
  const int n[3] = {nx, ny, nz};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float U = __fmul_rn((float)(uint32_t)(z[k] >> 40), 5.9604644775390625e-08f);  // exact
    t[k] = __fmul_rn((float)(n[k] - 1), __fadd_rn(0.1f, __fmul_rn(0.8f, U)));
  }
  const float2 ca = trig[(int)((z[3] >> 32) % 360u)];
  const float2 cb = trig[(int)((z[4] >> 32) % 360u)];
  const float2 cg = trig[(int)((z[5] >> 32) % 360u)];
  const float Rx[9] = {1.f, 0.f, 0.f, 0.f, ca.x, -ca.y, 0.f, ca.y, ca.x};
  const float Ry[9] = {cb.x, 0.f, cb.y, 0.f, 1.f, 0.f, -cb.y, 0.f, cb.x};
  const float Rz[9] = {cg.x, -cg.y, 0.f, cg.y, cg.x, 0.f, 0.f, 0.f, 1.f};
  float Ryx[9], R0[9];
  matmul3(Ry, Rx, Ryx);
  matmul3(Rz, Ryx, R0);
#pragma unroll
  for (int k = 0; k < 9; ++k) R0s[k] = __fmul_rn(R0[k], inv_s);
}

// ---- P6: alignment pose (ix, iy) of a restart, x rotation first then y (Alg. 1 lines 4-6):
//   R' = Rx(ax) (x) R0s,  v = R' d  (v_k = fma(R'_k2,d.z, fma(R'_k1,d.y, R'_k0*d.x)))
//   u_x = fma(sy, v_z, fma(cy, v_x, t_x)),  u_y = v_y + t_y,  u_z = fma(cy, v_z, fma(-sy, v_x, t_z))
// i.e. u = Ry(ay) (Rx(ax) (R0s d)) + t; u_y does not depend on ay.
__device__ __forceinline__ void align_rx(float2 cx_sx, const float *R0s, float *Rp) {
  const float Rx[9] = {1.f, 0.f, 0.f, 0.f, cx_sx.x, -cx_sx.y, 0.f, cx_sx.y, cx_sx.x};
  matmul3(Rx, R0s, Rp);
}
__device__ __forceinline__ float3 align_v(const float *Rp, float dx, float dy, float dz) {
  float3 v;
  v.x = __fmaf_rn(Rp[2], dz, __fmaf_rn(Rp[1], dy, __fmul_rn(Rp[0], dx)));
  v.y = __fmaf_rn(Rp[5], dz, __fmaf_rn(Rp[4], dy, __fmul_rn(Rp[3], dx)));
  v.z = __fmaf_rn(Rp[8], dz, __fmaf_rn(Rp[7], dy, __fmul_rn(Rp[6], dx)));
  return v;
}
__device__ __forceinline__ float3 align_u(float3 v, float cy, float sy, const float *t) {
  float3 u;
  u.x = __fmaf_rn(sy, v.z, __fmaf_rn(cy, v.x, t[0]));
  u.y = __fadd_rn(v.y, t[1]);
  u.z = __fmaf_rn(cy, v.z, __fmaf_rn(-sy, v.x, t[2]));
  return u;
}

// ---- P8: torsion rotation (Rodrigues) about unit axis k by table angle (c, s)
__device__ __forceinline__ void torsion_matrix(float kx, float ky, float kz, float c, float s, float *R) {
  const float C = __fsub_rn(1.0f, c);
  const float Ckx = __fmul_rn(C, kx), Cky = __fmul_rn(C, ky), Ckz = __fmul_rn(C, kz);
  const float skx = __fmul_rn(s, kx), sky = __fmul_rn(s, ky), skz = __fmul_rn(s, kz);
  R[0] = __fmaf_rn(Ckx, kx, c);
  R[1] = __fmaf_rn(Ckx, ky, -skz);
  R[2] = __fmaf_rn(Ckx, kz, sky);
  R[3] = __fmaf_rn(Cky, kx, skz);
  R[4] = __fmaf_rn(Cky, ky, c);
  R[5] = __fmaf_rn(Cky, kz, -skx);
  R[6] = __fmaf_rn(Ckz, kx, -sky);
  R[7] = __fmaf_rn(Ckz, ky, skx);
  R[8] = __fmaf_rn(Ckz, kz, c);
}

// p' = R (p - a) + a
__device__ __forceinline__ float3 torsion_apply(const float *R, float3 a, float px, float py, float pz) {
  const float wx = __fsub_rn(px, a.x), wy = __fsub_rn(py, a.y), wz = __fsub_rn(pz, a.z);
  float3 o;
  o.x = __fmaf_rn(R[2], wz, __fmaf_rn(R[1], wy, __fmaf_rn(R[0], wx, a.x)));
  o.y = __fmaf_rn(R[5], wz, __fmaf_rn(R[4], wy, __fmaf_rn(R[3], wx, a.y)));
  o.z = __fmaf_rn(R[8], wz, __fmaf_rn(R[7], wy, __fmaf_rn(R[6], wx, a.z)));
  return o;
}

// ---- P9: squared distance fma(dz,dz, fma(dy,dy, dx*dx))
__device__ __forceinline__ float dist2(float ax, float ay, float az, float bx, float by, float bz) {
  const float dx = __fsub_rn(ax, bx), dy = __fsub_rn(ay, by), dz = __fsub_rn(az, bz);
  return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

// ---- Blackwell packed f32x2 arithmetic (FFMA2 / FADD2): two IEEE round-to-nearest operations
// per instruction, each lane of the pair bit-identical to the scalar __fmaf_rn / __fadd_rn ----
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(f2_t v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t f2_sub(f2_t a, f2_t b) {
  f2_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
  f2_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// The per-function dynamic shared-memory limit is process-wide state: contexts on concurrent host
// threads launching one kernel with different sizes would race on it (a launch after another
// thread lowered it fails with "too many resources"), so it is always raised to the device's
// opt-in maximum; every launch still passes its own size.
inline void allow_max_smem(const void *func) {
  static const int max_smem = [] {
    int d = 0, v = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
    return v;
  }();
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, func) != cudaSuccess) return;
  cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem - (int)fa.sharedSizeBytes);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- bulk async copies (TMA engine, no tensor map) into shared memory, completion on an mbarrier ----
__device__ __forceinline__ unsigned smem_addr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
// make the initialised barriers visible to the async (bulk-copy) proxy
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
// dst, src 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
// the same copy into the same shared-memory offset of every CTA in mask (thread-block cluster);
// each destination's mbarrier at bar's offset receives the complete_tx
__device__ __forceinline__ void bulk_g2s_multicast(void *dst, const void *src, unsigned bytes, unsigned long long *bar,
                                                   unsigned mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "h"((unsigned short)mask)
      : "memory");
}
// the spin loop is C++ around one try_wait, so the compiler sees the loop
__device__ __forceinline__ bool mbar_try(unsigned long long *bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0u;
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
  while (!mbar_try(bar, parity)) {
  }
}
// CTA barrier without the .aligned requirement (threads of a warp may arrive from divergent
// paths, e.g. right after an mbarrier spin loop)
__device__ __forceinline__ void cta_sync_unaligned() { asm volatile("barrier.sync 0;" ::: "memory"); }

}  // namespace ds
