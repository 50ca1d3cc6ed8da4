// Device-side ingest: the synthetic ligand generator (SPEC.md:443-451
// generate_dataset; host version ds_generate_ligands in ds_host.cpp) and the packer
// (ds_pack_ligands) fused into one kernel that writes docking-ready device arrays — the packed
// atoms (xyz - c0, type), the fragment descriptors and the id hashes — so a screen shard is
// generated where it is docked instead of being built on the host and copied over PCIe.
//
// Warp per ligand.  Every operation is the host's, in the host's order, with explicit IEEE
// double rounding (__dadd_rn / __dmul_rn / __ddiv_rn / __dsqrt_rn: no contraction whatever the
// compiler flags) and the same SplitMix64 streams, so the arrays are bit-identical to
// generate_batch + pack on the host (GPU test).
#include <stdint.h>

#include "ds_kernels.cuh"

namespace ds {
namespace {

constexpr uint64_t kGold = 0x9E3779B97F4A7C15ull;
enum : uint64_t { kStHydro = 2, kStGeom = 3, kStFrag = 4 };

__device__ __forceinline__ uint64_t mix64d(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct DevRng {  // the host's Rng (ds_host.cpp), same constants
  uint64_t x;
  __device__ DevRng(uint64_t seed, uint64_t stream, uint64_t index)
      : x(mix64d(seed * kGold ^ mix64d(stream + 0x632BE59BD9B4E019ull)) + index * 0xD1B54A32D192ED03ull) {}
  __device__ uint64_t next() {
    x += kGold;
    return mix64d(x);
  }
  __device__ double u01() { return __dmul_rn((double)(next() >> 11), 1.0 / 9007199254740992.0); }
  __device__ uint32_t below(uint32_t n) { return (uint32_t)((next() >> 32) % n); }
  __device__ void unit(double v[3]) {
    for (;;) {
      const double x = __dsub_rn(__dmul_rn(2.0, u01()), 1.0);
      const double y = __dsub_rn(__dmul_rn(2.0, u01()), 1.0);
      const double z = __dsub_rn(__dmul_rn(2.0, u01()), 1.0);
      const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z));
      if (r2 > 1e-6 && r2 <= 1.0) {
        const double r = __dsqrt_rn(r2);
        v[0] = __ddiv_rn(x, r);
        v[1] = __ddiv_rn(y, r);
        v[2] = __ddiv_rn(z, r);
        return;
      }
    }
  }
};

__device__ __forceinline__ double ddist2(const double *a, const double *b) {
  const double dx = __dsub_rn(a[0], b[0]), dy = __dsub_rn(a[1], b[1]), dz = __dsub_rn(a[2], b[2]);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// FNV-1a 64 (ds_ligand_id_hash) over the decimal digits of v ("%lld")
__device__ __forceinline__ uint64_t fnv_decimal(uint64_t h, long long v) {
  char d[24];
  int n = 0;
  unsigned long long u = v < 0 ? 0ull - (unsigned long long)v : (unsigned long long)v;
  do {
    d[n++] = (char)('0' + (int)(u % 10ull));
    u /= 10ull;
  } while (u);
  if (v < 0) {
    h ^= (uint8_t)'-';
    h *= 0x100000001B3ull;
  }
  while (n) {
    h ^= (uint8_t)d[--n];
    h *= 0x100000001B3ull;
  }
  return h;
}

// hash of the generated id "lig_<seed>_<index>" (ds_generated_id)
__device__ __forceinline__ uint64_t generated_id_hash(long long seed, long long index) {
  uint64_t h = 0xCBF29CE484222325ull;
  const char pre[4] = {'l', 'i', 'g', '_'};
  for (int i = 0; i < 4; ++i) {
    h ^= (uint8_t)pre[i];
    h *= 0x100000001B3ull;
  }
  h = fnv_decimal(h, seed);
  h ^= (uint8_t)'_';
  h *= 0x100000001B3ull;
  return fnv_decimal(h, index);
}

constexpr int kGenWarps = 4;

// warp per ligand: the RNG stream is sequential, so every lane draws the same numbers (uniform
// control flow, no shuffles) and the O(A^2) distance checks of each candidate are split over the
// lanes (__all_sync gives the host's AND over all earlier atoms); positions live in shared memory
__global__ void __launch_bounds__(kGenWarps * 32)
    k_generate_ligands(long long seed, long long first_index, int count, const int2 *shapes, const int *atom_off,
                       const int *frag_off, float4 *atoms, uint32_t *frag_desc, uint64_t *id_hash) {
  __shared__ double s_pos[kGenWarps][DS_MAX_ATOMS][3];
  __shared__ uint8_t s_parent[kGenWarps][DS_MAX_ATOMS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double(*pos)[3] = s_pos[warp];
  uint8_t *parent = s_parent[warp];
  for (int i = blockIdx.x * kGenWarps + warp; i < count; i += gridDim.x * kGenWarps) {
    const long long gi = first_index + i;
    const int heavy = shapes[i].x, frags = shapes[i].y;
    // hydrogens per heavy atom (hydrogen_counts): counts re-derived on the fly below
    DevRng hr((uint64_t)seed, kStHydro, (uint64_t)gi);
    DevRng g((uint64_t)seed, kStGeom, (uint64_t)gi);
    // heavy chain: self-avoiding 1.5 Å steps (min 1.4 Å to every earlier non-neighbour)
    if (lane == 0) {
      pos[0][0] = pos[0][1] = pos[0][2] = 0.0;
      parent[0] = 0;
    }
    __syncwarp();
    for (int k = 1; k < heavy; ++k) {
      double cand[3];
      for (int attempt = 0; attempt < 64; ++attempt) {
        double u[3];
        g.unit(u);
        for (int c = 0; c < 3; ++c) cand[c] = __dadd_rn(pos[k - 1][c], __dmul_rn(1.5, u[c]));
        bool ok = true;
        for (int j = lane; j + 1 < k && ok; j += 32) ok = ddist2(cand, pos[j]) >= 1.4 * 1.4;
        if (__all_sync(kFull, ok)) break;
      }
      if (lane == 0) {
        for (int c = 0; c < 3; ++c) pos[k][c] = cand[c];
        parent[k] = (uint8_t)(k - 1);
      }
      __syncwarp();
    }
    // hydrogens at 1.0 Å from their heavy atom, >= 0.9 Å from every other atom if possible
    int a = heavy;
    for (int k = 0; k < heavy; ++k) {
      const int want = 1 + (int)(hr.next() & 1);
      const int room = DS_MAX_ATOMS - a;
      int nh = want < room ? want : room;
      if (nh < 0) nh = 0;
      for (int h = 0; h < nh; ++h, ++a) {
        double cand[3];
        for (int attempt = 0; attempt < 16; ++attempt) {
          double u[3];
          g.unit(u);
          for (int c = 0; c < 3; ++c) cand[c] = __dadd_rn(pos[k][c], __dmul_rn(1.0, u[c]));
          bool ok = true;
          for (int j = lane; j < a && ok; j += 32)
            if (j != k) ok = ddist2(cand, pos[j]) >= 0.9 * 0.9;
          if (__all_sync(kFull, ok)) break;
        }
        if (lane == 0) {
          for (int c = 0; c < 3; ++c) pos[a][c] = cand[c];
          parent[a] = (uint8_t)k;
        }
        __syncwarp();
      }
    }
    const int total = a;
    // pack (ds_pack_ligands): c0 = f32(f64 sequential mean of the f32 coordinates), d = p - c0
    double s[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < total; ++k)
      for (int c = 0; c < 3; ++c) s[c] = __dadd_rn(s[c], (double)__double2float_rn(pos[k][c]));
    float c0[3];
    for (int c = 0; c < 3; ++c) c0[c] = __double2float_rn(__ddiv_rn(s[c], (double)total));
    const int ao = atom_off[i];
    for (int k = 0; k < total; ++k) {
      const uint8_t t = k < heavy ? (uint8_t)(1 + g.below(DS_N_TYPES - 1)) : (uint8_t)0;
      if ((k & 31) == lane)
        atoms[ao + k] = make_float4(__fsub_rn(__double2float_rn(pos[k][0]), c0[0]),
                                    __fsub_rn(__double2float_rn(pos[k][1]), c0[1]),
                                    __fsub_rn(__double2float_rn(pos[k][2]), c0[2]), (float)t);
    }
    // rotatable bonds: F distinct chain bonds (k, k+1), k in [0, heavy-3], ascending; the moving
    // side is the tail component minus axis_end
    DevRng fr((uint64_t)seed, kStFrag, (uint64_t)gi);
    uint8_t cb[DS_MAX_ATOMS];
    const int nb = heavy - 2;
    for (int k = 0; k < nb; ++k) cb[k] = (uint8_t)k;
    for (int f = 0; f < frags; ++f) {  // partial Fisher-Yates
      const int j = f + (int)fr.below((uint32_t)(nb - f));
      const uint8_t t = cb[f];
      cb[f] = cb[j];
      cb[j] = t;
    }
    for (int f = 1; f < frags; ++f) {  // insertion sort (distinct keys: the same order as std::sort)
      const uint8_t v = cb[f];
      int j = f - 1;
      while (j >= 0 && cb[j] > v) {
        cb[j + 1] = cb[j];
        --j;
      }
      cb[j + 1] = v;
    }
    const int fo = frag_off[i];
    for (int f = 0; f < frags; ++f) {
      const int k = cb[f];
      uint32_t m[DS_MASK_WORDS];
#pragma unroll
      for (int w = 0; w < DS_MASK_WORDS; ++w) {
        const int t = 32 * w + lane;
        bool mv = false;
        if (t < total) {
          const int root = t < heavy ? t : parent[t];
          mv = root >= k + 1 && t != k + 1;
        }
        m[w] = __ballot_sync(kFull, mv);
      }
      if (lane == 0) {
        uint4 *d = reinterpret_cast<uint4 *>(frag_desc + (size_t)DS_FRAG_WORDS * (fo + f));
        d[0] = make_uint4(m[0], m[1], m[2], m[3]);
        d[1] = make_uint4(m[4], (uint32_t)k | ((uint32_t)(k + 1) << 8), 0u, 0u);
      }
    }
    if (lane == 0) id_hash[i] = generated_id_hash(seed, gi);
    __syncwarp();  // the next ligand overwrites pos / parent
  }
}

}  // namespace

void launch_generate_ligands(long long seed, long long first_index, int count, const int *shapes, const int *atom_off,
                             const int *frag_off, float4 *atoms, uint32_t *frag_desc, uint64_t *id_hash, int sm_count,
                             cudaStream_t st) {
  if (count <= 0) return;
  const int want = (count + kGenWarps - 1) / kGenWarps, cap = sm_count * 32;
  const int blocks = want < cap ? want : cap;
  k_generate_ligands<<<blocks, kGenWarps * 32, 0, st>>>(seed, first_index, count, reinterpret_cast<const int2 *>(shapes), atom_off,
                                            frag_off, atoms, frag_desc, id_hash);
}

}  // namespace ds
