// Host-side input makers and packing for libdockscreen (not on the timed path).
//
//  * ds_generate_ligands  — SPEC.md:443-451 generate_dataset (chain ligands, 1-2 H per
//                           heavy atom, self-avoiding 1.5 Å steps, F rotatable bonds).
//  * ds_build_pocket_grid — SPEC.md:453-461 build_pocket (shell-reward integer grid).
//  * ds_pack_ligands      — validation + the packed SoA batch layout.
//
// All randomness is a counter-based SplitMix64 keyed by (seed, global ligand index), so any
// shard of a 10M-ligand screen can be generated independently on its own rank
// (BASELINE config 5).  Only IEEE +,-,*,/,sqrt are used (no libm transcendental), so
// the generated inputs are identical on every x86-64 host.
#include "../../include/dockscreen.h"

#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdio.h>
#include <string.h>

#include <errno.h>
#include <stdlib.h>

#include <algorithm>
#include <charconv>
#include <string>
#include <vector>

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Rng {  // SplitMix64 stream
  uint64_t x;
  Rng(uint64_t seed, uint64_t stream, uint64_t index)
      : x(mix64(seed * kGolden ^ mix64(stream + 0x632BE59BD9B4E019ull)) + index * 0xD1B54A32D192ED03ull) {}
  uint64_t next() { x += kGolden; return mix64(x); }
  double u01() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
  uint32_t below(uint32_t n) { return (uint32_t)((next() >> 32) % n); }
  void unit(double v[3]) {  // rejection-sampled unit vector (no trig)
    for (;;) {
      double x = 2.0 * u01() - 1.0, y = 2.0 * u01() - 1.0, z = 2.0 * u01() - 1.0;
      double r2 = x * x + y * y + z * z;
      if (r2 > 1e-6 && r2 <= 1.0) {
        double r = sqrt(r2);
        v[0] = x / r; v[1] = y / r; v[2] = z / r;
        return;
      }
    }
  }
};

enum : uint64_t { kStreamShape = 1, kStreamHydro = 2, kStreamGeom = 3, kStreamFrag = 4, kStreamPocket = 5,
                  kStreamTable = 6 };

inline double dist2(const double *a, const double *b) {
  double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return dx * dx + dy * dy + dz * dz;
}

// number of hydrogens per heavy atom (1-2, total capped at DS_MAX_ATOMS)
int hydrogen_counts(int64_t seed, int64_t gi, int heavy, int *nh) {
  Rng r((uint64_t)seed, kStreamHydro, (uint64_t)gi);
  int total = heavy;
  for (int k = 0; k < heavy; ++k) {
    int want = 1 + (int)(r.next() & 1);
    int room = DS_MAX_ATOMS - total;
    int h = want < room ? want : room;
    if (h < 0) h = 0;
    if (nh) nh[k] = h;
    total += h;
  }
  return total;
}

thread_local char g_err[256];

}  // namespace

extern "C" {

uint64_t ds_ligand_id_hash(const char *id, size_t len) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (size_t i = 0; i < len; ++i) {
    h ^= (uint8_t)id[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

int ds_generated_id(int64_t seed, int64_t index, char *buf, size_t cap) {
  return snprintf(buf, cap, "lig_%lld_%lld", (long long)seed, (long long)index);
}

// ids first_index .. first_index + count - 1 as one byte blob + offsets (off[count] = total):
// with buf == NULL only the offsets are filled (size query); both passes OpenMP-parallel
// "%lld" of v into out (no terminator); returns the length
static int fmt_i64(int64_t v, char *out) {
  char tmp[24];
  int n = 0;
  uint64_t u = v < 0 ? (uint64_t)0 - (uint64_t)v : (uint64_t)v;
  do {
    tmp[n++] = (char)('0' + u % 10u);
    u /= 10u;
  } while (u);
  int k = 0;
  if (v < 0) out[k++] = '-';
  while (n) out[k++] = tmp[--n];
  return k;
}

// "lig_<seed>_<index>" (the snprintf format of ds_generated_id) into out; returns the length
static int fmt_generated_id(int64_t seed, int64_t index, char *out) {
  memcpy(out, "lig_", 4);
  int k = 4 + fmt_i64(seed, out + 4);
  out[k++] = '_';
  return k + fmt_i64(index, out + k);
}

int ds_generated_ids(int64_t seed, int64_t first_index, int32_t count, char *buf, int64_t *off) {
  if (count < 0 || !off) return DS_ERR_INVALID_ARG;
  std::vector<int32_t> len((size_t)count);
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < count; ++i) {
    char tmp[64];
    len[i] = fmt_generated_id(seed, first_index + i, tmp);
  }
  off[0] = 0;
  for (int32_t i = 0; i < count; ++i) off[i + 1] = off[i] + len[i];
  if (buf) {
#pragma omp parallel for schedule(static)
    for (int32_t i = 0; i < count; ++i) fmt_generated_id(seed, first_index + i, buf + off[i]);
  }
  return DS_OK;
}

int ds_mixed_shapes(int64_t seed, int64_t first_index, int32_t count, int32_t heavy_min, int32_t heavy_max,
                    int32_t frag_max, int32_t *shapes) {
  if (count < 0 || !shapes || heavy_min < 1 || heavy_max < heavy_min || heavy_max > DS_MAX_ATOMS || frag_max < 0)
    return DS_ERR_INVALID_ARG;
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < count; ++i) {
    Rng r((uint64_t)seed, kStreamShape, (uint64_t)(first_index + i));
    int heavy = heavy_min + (int)r.below((uint32_t)(heavy_max - heavy_min + 1));
    int fcap = std::min(frag_max, std::max(heavy - 2, 0));
    int frags = (int)r.below((uint32_t)(fcap + 1));
    shapes[2 * i] = heavy;
    shapes[2 * i + 1] = frags;
  }
  return DS_OK;
}

int ds_generate_ligands(int64_t seed, int64_t first_index, int32_t count, const int32_t *shapes,
                        int32_t *atom_off, int32_t *bond_off, int32_t *frag_off, float *atom_xyz,
                        uint8_t *atom_type, int32_t *bonds, int32_t *frag_axis, uint32_t *frag_mask) {
  if (count < 0 || !shapes || !atom_off || !bond_off || !frag_off) return DS_ERR_INVALID_ARG;
  for (int32_t i = 0; i < count; ++i) {
    int heavy = shapes[2 * i], frags = shapes[2 * i + 1];
    // InfeasibleShape: fragments >= heavy - 1, or the atom cap
    if (heavy < 1 || heavy > DS_MAX_ATOMS || frags < 0 || (frags > 0 && frags >= heavy - 1)) return DS_ERR_INFEASIBLE_SHAPE;
  }
  if (!atom_xyz) {  // pass 1: sizes
    std::vector<int> tot(count);
#pragma omp parallel for schedule(static)
    for (int32_t i = 0; i < count; ++i) tot[i] = hydrogen_counts(seed, first_index + i, shapes[2 * i], nullptr);
    atom_off[0] = bond_off[0] = frag_off[0] = 0;
    for (int32_t i = 0; i < count; ++i) {
      atom_off[i + 1] = atom_off[i] + tot[i];
      bond_off[i + 1] = bond_off[i] + tot[i] - 1;
      frag_off[i + 1] = frag_off[i] + shapes[2 * i + 1];
    }
    return DS_OK;
  }
  if (!atom_type || !bonds || !frag_axis || !frag_mask) return DS_ERR_INVALID_ARG;
#pragma omp parallel for schedule(dynamic, 64)
  for (int32_t i = 0; i < count; ++i) {
    const int64_t gi = first_index + i;
    const int heavy = shapes[2 * i], frags = shapes[2 * i + 1];
    int nh[DS_MAX_ATOMS];
    const int total = hydrogen_counts(seed, gi, heavy, nh);
    double pos[DS_MAX_ATOMS][3];
    int parent[DS_MAX_ATOMS];
    Rng g((uint64_t)seed, kStreamGeom, (uint64_t)gi);
    // heavy chain: self-avoiding 1.5 Å steps (min 1.4 Å to every earlier non-neighbour)
    pos[0][0] = pos[0][1] = pos[0][2] = 0.0;
    parent[0] = -1;
    for (int k = 1; k < heavy; ++k) {
      double cand[3];
      for (int attempt = 0; attempt < 64; ++attempt) {
        double u[3];
        g.unit(u);
        for (int c = 0; c < 3; ++c) cand[c] = pos[k - 1][c] + 1.5 * u[c];
        bool ok = true;
        for (int j = 0; j + 1 < k && ok; ++j) ok = dist2(cand, pos[j]) >= 1.4 * 1.4;
        if (ok) break;
      }
      for (int c = 0; c < 3; ++c) pos[k][c] = cand[c];
      parent[k] = k - 1;
    }
    // hydrogens at 1.0 Å from their heavy atom, >= 0.9 Å from every other atom if possible
    int a = heavy;
    for (int k = 0; k < heavy; ++k) {
      for (int h = 0; h < nh[k]; ++h, ++a) {
        double cand[3];
        for (int attempt = 0; attempt < 16; ++attempt) {
          double u[3];
          g.unit(u);
          for (int c = 0; c < 3; ++c) cand[c] = pos[k][c] + 1.0 * u[c];
          bool ok = true;
          for (int j = 0; j < a && ok; ++j)
            if (j != k) ok = dist2(cand, pos[j]) >= 0.9 * 0.9;
          if (ok) break;
        }
        for (int c = 0; c < 3; ++c) pos[a][c] = cand[c];
        parent[a] = k;
      }
    }
    const int ao = atom_off[i];
    for (int k = 0; k < total; ++k) {
      for (int c = 0; c < 3; ++c) atom_xyz[3 * (ao + k) + c] = (float)pos[k][c];
      atom_type[ao + k] = k < heavy ? (uint8_t)(1 + g.below(DS_N_TYPES - 1)) : (uint8_t)0;
    }
    // bonds: chain then X-H, in atom order of the child
    const int bo = bond_off[i];
    for (int k = 1; k < total; ++k) {
      bonds[2 * (bo + k - 1)] = parent[k];
      bonds[2 * (bo + k - 1) + 1] = k;
    }
    // rotatable bonds: F distinct chain bonds (k, k+1) with k in [0, heavy-3], ascending;
    // the moving side is the tail component minus axis_end (DESIGN.md §3 P13)
    Rng fr((uint64_t)seed, kStreamFrag, (uint64_t)gi);
    int cand_bonds[DS_MAX_ATOMS];
    const int nb = heavy - 2;
    for (int k = 0; k < nb; ++k) cand_bonds[k] = k;
    for (int f = 0; f < frags; ++f) {  // partial Fisher-Yates
      int j = f + (int)fr.below((uint32_t)(nb - f));
      std::swap(cand_bonds[f], cand_bonds[j]);
    }
    std::sort(cand_bonds, cand_bonds + frags);
    const int fo = frag_off[i];
    for (int f = 0; f < frags; ++f) {
      const int k = cand_bonds[f];
      frag_axis[2 * (fo + f)] = k;
      frag_axis[2 * (fo + f) + 1] = k + 1;
      uint32_t *m = frag_mask + (size_t)DS_MASK_WORDS * (fo + f);
      for (int w = 0; w < DS_MASK_WORDS; ++w) m[w] = 0;
      for (int t = 0; t < total; ++t) {
        const int root = t < heavy ? t : parent[t];
        if (root >= k + 1 && t != k + 1) m[t >> 5] |= 1u << (t & 31);
      }
    }
  }
  return DS_OK;
}

int ds_pack_ligands(int32_t count, const int32_t *atom_off, const float *atom_xyz, const uint8_t *atom_type,
                    const int32_t *frag_off, const int32_t *frag_axis, const uint32_t *frag_mask, const char *ids,
                    const int64_t *id_off, float *atom_xyzt, uint32_t *frag_desc, uint64_t *id_hash, float *centroid,
                    int32_t *bad_index) {
  if (count < 0 || !atom_off || !atom_xyz || !atom_type || !frag_off || !atom_xyzt || !frag_desc || !id_hash)
    return DS_ERR_INVALID_ARG;
  int first_bad = -1, first_code = DS_OK;
#pragma omp parallel for schedule(static)
  for (int32_t i = 0; i < count; ++i) {
    const int a0 = atom_off[i], A = atom_off[i + 1] - a0;
    int code = DS_OK;
    if (A < 1) code = DS_ERR_INVALID_ARG;
    else if (A > DS_MAX_ATOMS) code = DS_ERR_TOO_MANY_ATOMS;
    for (int k = 0; k < A && code == DS_OK; ++k)
      if (atom_type[a0 + k] >= DS_N_TYPES) code = DS_ERR_INDEX_OUT_OF_RANGE;
    for (int f = frag_off[i]; f < frag_off[i + 1] && code == DS_OK; ++f) {
      const int b = frag_axis[2 * f], e = frag_axis[2 * f + 1];
      if (b < 0 || e < 0 || b >= A || e >= A) { code = DS_ERR_INDEX_OUT_OF_RANGE; break; }
      const uint32_t *m = frag_mask + (size_t)DS_MASK_WORDS * f;
      int pop = 0;
      for (int w = 0; w < DS_MASK_WORDS; ++w) {
        uint32_t valid = (A >= 32 * (w + 1)) ? 0xFFFFFFFFu : (A <= 32 * w ? 0u : ((1u << (A - 32 * w)) - 1u));
        if (m[w] & ~valid) { code = DS_ERR_INDEX_OUT_OF_RANGE; break; }
        pop += __builtin_popcount(m[w]);
      }
      if (code != DS_OK) break;
      const bool b_in = (m[b >> 5] >> (b & 31)) & 1, e_in = (m[e >> 5] >> (e & 31)) & 1;
      // axis atoms distinct and outside the mask; mask non-empty proper subset
      if (b == e || b_in || e_in || pop == 0 || pop > A - 2) code = DS_ERR_MALFORMED_FRAGMENT;
    }
    if (code != DS_OK) {
#pragma omp critical
      {
        if (first_bad < 0 || i < first_bad) { first_bad = i; first_code = code; }
      }
      continue;
    }
    // c0 = f32(f64 sequential mean), d = f32(p - c0)   (DESIGN.md §3 P2)
    double s[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < A; ++k)
      for (int c = 0; c < 3; ++c) s[c] += (double)atom_xyz[3 * (a0 + k) + c];
    float c0[3];
    for (int c = 0; c < 3; ++c) c0[c] = (float)(s[c] / (double)A);
    for (int k = 0; k < A; ++k) {
      float *o = atom_xyzt + 4 * (size_t)(a0 + k);
      for (int c = 0; c < 3; ++c) o[c] = atom_xyz[3 * (a0 + k) + c] - c0[c];
      o[3] = (float)atom_type[a0 + k];
    }
    if (centroid)
      for (int c = 0; c < 3; ++c) centroid[3 * i + c] = c0[c];
    for (int f = frag_off[i]; f < frag_off[i + 1]; ++f) {
      uint32_t *d = frag_desc + (size_t)DS_FRAG_WORDS * f;
      for (int w = 0; w < DS_MASK_WORDS; ++w) d[w] = frag_mask[(size_t)DS_MASK_WORDS * f + w];
      d[5] = (uint32_t)frag_axis[2 * f] | ((uint32_t)frag_axis[2 * f + 1] << 8);
      d[6] = d[7] = 0;
    }
    if (ids) id_hash[i] = ds_ligand_id_hash(ids + id_off[i], (size_t)(id_off[i + 1] - id_off[i]));
  }
  if (first_bad >= 0) {
    if (bad_index) *bad_index = first_bad;
    return first_code;
  }
  return DS_OK;
}

int ds_generate_pocket_atoms(int64_t seed, int32_t n, float rmin, float rmax, float *atom_xyz, uint8_t *atom_type) {
  if (n < 0 || !atom_xyz || !atom_type || !(rmax > 0) || rmin < 0 || rmin > rmax) return DS_ERR_INVALID_ARG;
  Rng r((uint64_t)seed, kStreamPocket, 0);
  const double lo2 = (double)rmin * rmin, hi2 = (double)rmax * rmax;
  for (int32_t i = 0; i < n; ++i) {
    double p[3];
    for (;;) {
      for (int c = 0; c < 3; ++c) p[c] = (2.0 * r.u01() - 1.0) * (double)rmax;
      double q = p[0] * p[0] + p[1] * p[1] + p[2] * p[2];
      if (q >= lo2 && q <= hi2) break;
    }
    for (int c = 0; c < 3; ++c) atom_xyz[3 * i + c] = (float)p[c];
    atom_type[i] = (uint8_t)(1 + r.below(DS_N_TYPES - 1));
  }
  return DS_OK;
}

int ds_build_pocket_grid(const float *atom_xyz, int32_t n_atoms, float spacing, float padding, float origin[3],
                         int32_t dims[3], int32_t *values) {
  if (n_atoms <= 0) return DS_ERR_EMPTY_POCKET;
  if (!atom_xyz || !(spacing > 0) || padding < 0 || !origin || !dims) return DS_ERR_INVALID_ARG;
  double lo[3], hi[3];
  for (int c = 0; c < 3; ++c) lo[c] = hi[c] = atom_xyz[c];
  for (int i = 1; i < n_atoms; ++i)
    for (int c = 0; c < 3; ++c) {
      lo[c] = std::min(lo[c], (double)atom_xyz[3 * i + c]);
      hi[c] = std::max(hi[c], (double)atom_xyz[3 * i + c]);
    }
  for (int c = 0; c < 3; ++c) {
    origin[c] = (float)(lo[c] - (double)padding);
    double span = (hi[c] + (double)padding) - (double)origin[c];
    dims[c] = (int32_t)ceil(span / (double)spacing - 1e-9) + 1;
    if (dims[c] < 1) dims[c] = 1;
  }
  if (!values) return DS_OK;
  const int nx = dims[0], ny = dims[1], nz = dims[2];
#pragma omp parallel for schedule(static) collapse(2)
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        const double node[3] = {(double)origin[0] + x * (double)spacing, (double)origin[1] + y * (double)spacing,
                                (double)origin[2] + z * (double)spacing};
        double best = INFINITY;
        for (int i = 0; i < n_atoms; ++i) {
          const double a[3] = {atom_xyz[3 * i], atom_xyz[3 * i + 1], atom_xyz[3 * i + 2]};
          best = std::min(best, dist2(node, a));
        }
        const double d = sqrt(best);
        // g(d): -1 at contact -> +1 at 3 Å, flat to 5 Å, -> -1 at 8 Å, -1 beyond (P18)
        double g;
        if (d <= 3.0) g = -1.0 + 2.0 * d / 3.0;
        else if (d <= 5.0) g = 1.0;
        else if (d <= 8.0) g = 1.0 - 2.0 * (d - 5.0) / 3.0;
        else g = -1.0;
        values[(size_t)x + (size_t)nx * ((size_t)y + (size_t)ny * z)] = (int32_t)nearbyint(10.0 * g);
      }
  return DS_OK;
}

// Gather / scatter of selected rows of a CSR array (the engines' per-bucket batches): rows sel[k]
// of src (offsets src_off, elem_bytes per element) become rows k of dst.  Pass 1 (dst == NULL)
// fills dst_off (n_sel + 1 entries); OpenMP over rows.
int ds_csr_gather(int32_t n_sel, const int32_t *sel, const int32_t *src_off, const void *src, int32_t elem_bytes,
                  int32_t *dst_off, void *dst) {
  if (n_sel < 0 || !sel || !src_off || !dst_off || elem_bytes <= 0) return DS_ERR_INVALID_ARG;
  if (!dst) {
    dst_off[0] = 0;
    for (int32_t k = 0; k < n_sel; ++k) dst_off[k + 1] = dst_off[k] + (src_off[sel[k] + 1] - src_off[sel[k]]);
    return DS_OK;
  }
  if (!src && dst_off[n_sel] > 0) return DS_ERR_INVALID_ARG;
#pragma omp parallel for schedule(static) if (n_sel >= 2048)
  for (int32_t k = 0; k < n_sel; ++k) {
    const int32_t i = sel[k];
    memcpy((char *)dst + (size_t)dst_off[k] * elem_bytes, (const char *)src + (size_t)src_off[i] * elem_bytes,
           (size_t)(src_off[i + 1] - src_off[i]) * elem_bytes);
  }
  return DS_OK;
}

// inverse: rows k of src (offsets src_off) go to rows sel[k] of dst (offsets dst_off)
int ds_csr_scatter(int32_t n_sel, const int32_t *sel, const int32_t *src_off, const void *src, int32_t elem_bytes,
                   const int32_t *dst_off, void *dst) {
  if (n_sel < 0 || !sel || !src_off || !dst_off || elem_bytes <= 0 || (!src && n_sel) || (!dst && n_sel))
    return DS_ERR_INVALID_ARG;
#pragma omp parallel for schedule(static) if (n_sel >= 2048)
  for (int32_t k = 0; k < n_sel; ++k) {
    const int32_t i = sel[k];
    memcpy((char *)dst + (size_t)dst_off[i] * elem_bytes, (const char *)src + (size_t)src_off[k] * elem_bytes,
           (size_t)(src_off[k + 1] - src_off[k]) * elem_bytes);
  }
  return DS_OK;
}

int ds_set_host_threads(int32_t n) {
  if (n < 1) return DS_ERR_INVALID_ARG;
  omp_set_num_threads(n);  // the calling thread's parallel regions (OpenMP nthreads-var is per thread)
  return DS_OK;
}

int ds_default_table(int64_t seed, float *table) {
  if (!table) return DS_ERR_INVALID_ARG;
  Rng r((uint64_t)seed, kStreamTable, 0);
  for (int i = 0; i < DS_N_TYPES; ++i)
    for (int j = i; j < DS_N_TYPES; ++j) {
      float w = (float)(2.0 * r.u01() - 1.0);
      table[i * DS_N_TYPES + j] = table[j * DS_N_TYPES + i] = w;
    }
  return DS_OK;
}

}  // extern "C"

// ---- native .ligq parser (io.parse_ligand_file restated) -------------------
// The text is cut at its MOL records; molecules are parsed and validated (validate_ligand,
// SPEC.md:81-89, including the bond-cut invariants) in parallel, then concatenated in file order.
// Semantics follow io.parse_ligand_file line for line: records are the first whitespace-separated
// token; a MOL id is the stripped line minus "MOL "; a molecule without END that is followed by
// another MOL is dropped; a non-empty line outside a molecule, a malformed record or a missing
// final END is a parse error; the first error in file order is reported.
namespace {

struct LigqMol {
  std::string id;
  std::vector<float> xyz;
  std::vector<uint8_t> type;
  std::vector<int32_t> bonds;   // pairs
  std::vector<int32_t> axis;    // pairs
  std::vector<uint32_t> mask;   // DS_MASK_WORDS per fragment
  int64_t line = 0;             // line of the MOL record
  int code = 0;                 // parse error before END (DS_ERR_PARSE) or validation DS_ERR_*
  int64_t err_line = 0;
  std::string err;
  bool ended = false;
  bool invalid = false;         // code is a validation error (the reference raises it at END)
  std::string trail_err;        // "record outside MOL" after END (reported after a validation error)
};

inline bool ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f'; }

// split [b, e) into tokens
int tokens(const char *b, const char *e, const char **tb, const char **te, int maxt) {
  int n = 0;
  while (b < e) {
    while (b < e && ws(*b)) ++b;
    if (b >= e) break;
    const char *s = b;
    while (b < e && !ws(*b)) ++b;
    if (n < maxt) {
      tb[n] = s;
      te[n] = b;
    }
    ++n;
  }
  return n;
}

bool tok_eq(const char *b, const char *e, const char *lit) {
  const size_t n = strlen(lit);
  return (size_t)(e - b) == n && memcmp(b, lit, n) == 0;
}

// Python int() / float() on one token (a leading '+' allowed, the whole token consumed); floats are
// parsed to the nearest double and rounded to f32, as float(np.float32(float(t)))
bool parse_int(const char *b, const char *e, long long *v) {
  if (b < e && *b == '+' && e - b > 1 && b[1] != '-') ++b;
  const auto r = std::from_chars(b, e, *v);
  return r.ec == std::errc() && r.ptr == e && b < e;
}

bool parse_f32(const char *b, const char *e, float *v) {
  if (b < e && *b == '+' && e - b > 1 && b[1] != '-') ++b;
  double x;
  const auto r = std::from_chars(b, e, x);
  if (r.ec != std::errc() || r.ptr != e || b == e) {
    // from_chars reports out-of-range values as errors; Python gives +-inf or a subnormal/0
    if (r.ec == std::errc::result_out_of_range && r.ptr == e) {
      std::string s(b, e);
      x = strtod(s.c_str(), nullptr);
    } else {
      return false;
    }
  }
  *v = (float)x;
  return true;
}

// validate_ligand over plain arrays, check for check in the reference's order;
// returns 0 or the DS_ERR_* code (why = the reference's message without the ligand id)
int validate_arrays(int n, const long long *type_raw, const uint8_t *heavy_flag, int nb, const int32_t *bonds, int nf,
                    const int32_t *axis, const int64_t *mv_off, const long long *mv, std::string *why) {
  if (n > DS_MAX_ATOMS) return *why = std::to_string(n) + " atoms > " + std::to_string(DS_MAX_ATOMS), DS_ERR_TOO_MANY_ATOMS;
  if (n < 1) return *why = "ligand has no atoms", DS_ERR_INDEX_OUT_OF_RANGE;
  for (int i = 0; i < n; ++i) {
    if (type_raw[i] < 0 || type_raw[i] >= DS_N_TYPES)
      return *why = "element_type " + std::to_string(type_raw[i]) + " outside 0..15", DS_ERR_INDEX_OUT_OF_RANGE;
    if ((bool)heavy_flag[i] != (type_raw[i] != 0)) return *why = "is_heavy inconsistent with element_type", DS_ERR_MALFORMED_FRAGMENT;
  }
  for (int k = 0; k < nb; ++k)
    if (bonds[2 * k] < 0 || bonds[2 * k] >= n || bonds[2 * k + 1] < 0 || bonds[2 * k + 1] >= n)
      return *why = "bond (" + std::to_string(bonds[2 * k]) + "," + std::to_string(bonds[2 * k + 1]) + ") out of range",
             DS_ERR_INDEX_OUT_OF_RANGE;
  std::vector<std::vector<int>> adj;
  for (int f = 0; f < nf; ++f) {
    const long long ab = axis[2 * f], ae = axis[2 * f + 1];
    if (!(0 <= ab && ab < n && 0 <= ae && ae < n)) return *why = "fragment axis out of range", DS_ERR_INDEX_OUT_OF_RANGE;
    for (int64_t k = mv_off[f]; k < mv_off[f + 1]; ++k)
      if (!(0 <= mv[k] && mv[k] < n)) return *why = "moving_mask index out of range", DS_ERR_INDEX_OUT_OF_RANGE;
    std::vector<char> inm(n, 0);
    int msize = 0;
    for (int64_t k = mv_off[f]; k < mv_off[f + 1]; ++k)
      if (!inm[mv[k]]) inm[mv[k]] = 1, ++msize;
    if (ab == ae || inm[ab] || inm[ae]) return *why = "axis atoms must be distinct and outside the mask", DS_ERR_MALFORMED_FRAGMENT;
    if (msize == 0 || msize >= n) return *why = "moving_mask must be a non-empty proper subset", DS_ERR_MALFORMED_FRAGMENT;
    bool is_bond = false;
    for (int k = 0; k < nb && !is_bond; ++k)
      is_bond = (bonds[2 * k] == ab && bonds[2 * k + 1] == ae) || (bonds[2 * k] == ae && bonds[2 * k + 1] == ab);
    if (!is_bond) return *why = "fragment axis is not a bond", DS_ERR_MALFORMED_FRAGMENT;
    if (adj.empty()) {
      adj.assign(n, {});
      for (int k = 0; k < nb; ++k) {
        adj[bonds[2 * k]].push_back(k);
        adj[bonds[2 * k + 1]].push_back(k);
      }
    }
    // connected components of the bond graph without every (ab, ae) / (ae, ab) bond
    std::vector<int> comp(n, -1), st;
    int nc = 0;
    for (int s0 = 0; s0 < n; ++s0) {
      if (comp[s0] >= 0) continue;
      st.assign(1, s0);
      comp[s0] = nc;
      while (!st.empty()) {
        const int u = st.back();
        st.pop_back();
        for (int k : adj[u]) {
          const int a2 = bonds[2 * k], b2 = bonds[2 * k + 1];
          if ((a2 == ab && b2 == ae) || (a2 == ae && b2 == ab)) continue;
          const int w = a2 == u ? b2 : a2;
          if (comp[w] < 0) comp[w] = nc, st.push_back(w);
        }
      }
      ++nc;
    }
    if (comp[ab] == comp[ae]) return *why = "removing the axis bond does not split the ligand", DS_ERR_MALFORMED_FRAGMENT;
    if (nc != 2) return *why = "cutting the axis bond must leave exactly two parts", DS_ERR_MALFORMED_FRAGMENT;
    bool side_b = true, side_e = true;
    for (int i = 0; i < n; ++i) {
      const bool pb = comp[i] == comp[ab] && i != ab && i != ae, pe = comp[i] == comp[ae] && i != ab && i != ae;
      if ((bool)inm[i] != pb) side_b = false;
      if ((bool)inm[i] != pe) side_e = false;
    }
    if (!side_b && !side_e) return *why = "moving_mask is not one side of the axis bond", DS_ERR_MALFORMED_FRAGMENT;
  }
  return DS_OK;
}

int validate_mol(const LigqMol &m, const std::vector<uint8_t> &heavy_flag, const std::vector<std::vector<long long>> &fr,
                 const std::vector<long long> &type_raw, std::string *why) {
  std::vector<int64_t> off(fr.size() + 1, 0);
  std::vector<long long> mv;
  for (size_t f = 0; f < fr.size(); ++f) {
    mv.insert(mv.end(), fr[f].begin(), fr[f].end());
    off[f + 1] = (int64_t)mv.size();
  }
  return validate_arrays((int)m.type.size(), type_raw.data(), heavy_flag.data(), (int)(m.bonds.size() / 2),
                         m.bonds.data(), (int)fr.size(), m.axis.data(), off.data(), mv.data(), why);
}

// parse one molecule: [b, e) starts at its MOL line (line number `line`)
void parse_mol(const char *b, const char *e, int64_t line, LigqMol *m) {
  m->line = line;
  std::vector<uint8_t> heavy;
  std::vector<long long> type_raw;
  std::vector<std::vector<long long>> fr;
  const char *p = b;
  int64_t ln = line;
  bool first = true;
  const char *tb[8], *te[8];
  auto perr = [&](const std::string &msg) {
    m->code = DS_ERR_PARSE;
    m->err_line = ln;
    m->err = "line " + std::to_string(ln) + ": " + msg;
  };
  while (p < e && !m->ended && !m->code) {
    const char *q = (const char *)memchr(p, '\n', (size_t)(e - p));
    const char *le = q ? q : e;
    const int nt = tokens(p, le, tb, te, 8);
    if (first) {  // the MOL record: id = stripped line minus "MOL "
      const char *s = p, *t = le;
      while (s < t && ws(*s)) ++s;
      while (t > s && ws(t[-1])) --t;
      m->id = t - s > 4 ? std::string(s + 4, t) : std::string();
      first = false;
    } else if (nt > 0) {
      if (tok_eq(tb[0], te[0], "ATOM")) {
        long long idx, typ;
        float x, y, z;
        if (nt < 7) return perr("list index out of range");
        if (!parse_int(tb[1], te[1], &idx) || !parse_int(tb[2], te[2], &typ)) return perr("invalid literal for int()");
        if (idx != (long long)m->type.size()) return perr("atom index " + std::to_string(idx) + " out of order");
        if (!parse_f32(tb[3], te[3], &x) || !parse_f32(tb[4], te[4], &y) || !parse_f32(tb[5], te[5], &z))
          return perr("could not convert string to float");
        m->xyz.insert(m->xyz.end(), {x, y, z});
        type_raw.push_back(typ);
        m->type.push_back((uint8_t)(typ & 0xFF));
        heavy.push_back(!tok_eq(tb[6], te[6], "H"));
      } else if (tok_eq(tb[0], te[0], "BOND")) {
        long long a, c;
        if (nt < 3) return perr("list index out of range");
        if (!parse_int(tb[1], te[1], &a) || !parse_int(tb[2], te[2], &c)) return perr("invalid literal for int()");
        m->bonds.push_back((int32_t)std::max(std::min(a, (long long)INT32_MAX), (long long)INT32_MIN));
        m->bonds.push_back((int32_t)std::max(std::min(c, (long long)INT32_MAX), (long long)INT32_MIN));
      } else if (tok_eq(tb[0], te[0], "FRAG")) {
        long long a, c;
        if (nt < 3) return perr("list index out of range");
        if (!parse_int(tb[1], te[1], &a) || !parse_int(tb[2], te[2], &c)) return perr("invalid literal for int()");
        std::vector<long long> mv;
        // the moving atoms: every token after the axis (re-tokenise, there may be many)
        const char *s = te[2];
        while (s < le) {
          while (s < le && ws(*s)) ++s;
          if (s >= le) break;
          const char *t = s;
          while (t < le && !ws(*t)) ++t;
          long long v;
          if (!parse_int(s, t, &v)) return perr("invalid literal for int()");
          mv.push_back(v);
          s = t;
        }
        m->axis.push_back((int32_t)std::max(std::min(a, (long long)INT32_MAX), (long long)INT32_MIN));
        m->axis.push_back((int32_t)std::max(std::min(c, (long long)INT32_MAX), (long long)INT32_MIN));
        fr.push_back(std::move(mv));
      } else if (tok_eq(tb[0], te[0], "END")) {
        m->ended = true;
      } else {
        return perr("unknown record '" + std::string(tb[0], te[0]) + "'");
      }
    }
    p = q ? q + 1 : e;
    ++ln;
  }
  if (!m->ended || m->code) return;
  // validated at END (the reference raises there, before it reads any later line)
  std::string why;
  const int v = validate_mol(*m, heavy, fr, type_raw, &why);
  if (v) {
    m->code = v;
    m->invalid = true;
    m->err_line = m->line;
    m->err = "molecule " + m->id + " (line " + std::to_string(m->line) + "): " + why;
  }
  // anything after END up to the next MOL must be blank ("record outside MOL")
  while (p < e) {
    const char *q = (const char *)memchr(p, '\n', (size_t)(e - p));
    const char *le = q ? q : e;
    if (tokens(p, le, tb, te, 1) > 0) {
      m->trail_err = "line " + std::to_string(ln) + ": record outside MOL";
      break;
    }
    p = q ? q + 1 : e;
    ++ln;
  }
  if (v) return;
  const int n = (int)m->type.size();
  m->mask.assign(fr.size() * DS_MASK_WORDS, 0u);
  for (size_t f = 0; f < fr.size(); ++f)
    for (long long v2 : fr[f]) m->mask[f * DS_MASK_WORDS + (v2 >> 5)] |= 1u << (v2 & 31);
  (void)n;
}

}  // namespace

struct ds_ligq {
  std::vector<LigqMol> mols;  // kept molecules, file order
  int64_t atoms = 0, bonds = 0, frags = 0, id_bytes = 0;
  int32_t skipped = 0;
};

extern "C" {

int ds_ligq_parse(const char *text, int64_t len, int32_t skip_invalid, ds_ligq **out, int64_t counts[6],
                  char *err, int32_t err_len) {
  if (!out || !counts || (!text && len > 0) || len < 0) return DS_ERR_INVALID_ARG;
  *out = nullptr;
  auto set_err = [&](const std::string &s) {
    if (err && err_len > 0) {
      strncpy(err, s.c_str(), (size_t)err_len - 1);
      err[err_len - 1] = 0;
    }
  };
  // MOL line starts: the text is cut into per-thread pieces at line boundaries, each piece scanned
  // for line heads (and newlines, for line numbers), then stitched in order
  int nthr = 1;
#ifdef _OPENMP
  nthr = std::max(1, std::min(omp_get_max_threads(), (int)(len / (1 << 20)) + 1));
#endif
  std::vector<int64_t> cut(nthr + 1);
  cut[0] = 0;
  cut[nthr] = len;
  for (int t = 1; t < nthr; ++t) {
    int64_t p = std::max(len * t / nthr, cut[t - 1]);
    const char *q = p < len ? (const char *)memchr(text + p, '\n', (size_t)(len - p)) : nullptr;
    cut[t] = q ? (q - text) + 1 : len;
  }
  std::vector<std::vector<int64_t>> pst(nthr), pln(nthr);
  std::vector<int64_t> nlines(nthr, 0), pre_nb(nthr, -1), pre_nb_ln(nthr, 0);
#pragma omp parallel for schedule(static, 1) num_threads(nthr)
  for (int t = 0; t < nthr; ++t) {
    int64_t ln = 0;
    for (int64_t p = cut[t]; p < cut[t + 1];) {
      const char *q = (const char *)memchr(text + p, '\n', (size_t)(cut[t + 1] - p));
      const int64_t le = q ? q - text : cut[t + 1];
      int64_t s2 = p;
      while (s2 < le && ws(text[s2])) ++s2;
      if (s2 < le) {
        int64_t e2 = s2;
        while (e2 < le && !ws(text[e2])) ++e2;
        if (e2 - s2 == 3 && memcmp(text + s2, "MOL", 3) == 0) {
          pst[t].push_back(p);
          pln[t].push_back(ln);
        } else if (pst[t].empty() && pre_nb[t] < 0) {
          pre_nb[t] = p;
          pre_nb_ln[t] = ln;
        }
      }
      p = q ? le + 1 : cut[t + 1];
      ++ln;
    }
    nlines[t] = ln;
  }
  std::vector<int64_t> starts, lines;
  int64_t base_ln = 1;
  for (int t = 0; t < nthr; ++t) {
    if (starts.empty() && pre_nb[t] >= 0) {  // a record before the first MOL
      set_err("line " + std::to_string(base_ln + pre_nb_ln[t]) + ": record outside MOL");
      return DS_ERR_PARSE;
    }
    for (size_t k = 0; k < pst[t].size(); ++k) {
      starts.push_back(pst[t][k]);
      lines.push_back(base_ln + pln[t][k]);
    }
    base_ln += nlines[t];
  }
  const int64_t nm = (int64_t)starts.size();
  std::vector<LigqMol> mols((size_t)nm);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t k = 0; k < nm; ++k)
    parse_mol(text + starts[k], text + (k + 1 < nm ? starts[k + 1] : len), lines[k], &mols[k]);
  ds_ligq *h = new ds_ligq();
  for (int64_t k = 0; k < nm; ++k) {
    LigqMol &m = mols[k];
    if (m.code == DS_ERR_PARSE) {
      set_err(m.err);
      delete h;
      return DS_ERR_PARSE;
    }
    if (!m.ended) {
      if (k + 1 == nm) {  // unterminated last molecule
        set_err("missing END");
        delete h;
        return DS_ERR_PARSE;
      }
      continue;  // the reference parser silently drops a molecule cut short by the next MOL
    }
    if (m.code) {
      if (!skip_invalid) {
        set_err(m.err);
        delete h;
        return m.code;
      }
      ++h->skipped;
    }
    if (!m.trail_err.empty()) {
      set_err(m.trail_err);
      delete h;
      return DS_ERR_PARSE;
    }
    if (m.code) continue;
    h->atoms += (int64_t)m.type.size();
    h->bonds += (int64_t)m.bonds.size() / 2;
    h->frags += (int64_t)m.axis.size() / 2;
    h->id_bytes += (int64_t)m.id.size();
    h->mols.push_back(std::move(m));
  }
  counts[0] = (int64_t)h->mols.size();
  counts[1] = h->atoms;
  counts[2] = h->bonds;
  counts[3] = h->frags;
  counts[4] = h->id_bytes;
  counts[5] = h->skipped;
  *out = h;
  return DS_OK;
}

int ds_ligq_fill(const ds_ligq *h, int32_t *atom_off, float *atom_xyz, uint8_t *atom_type, int32_t *bond_off,
                 int32_t *bonds, int32_t *frag_off, int32_t *frag_axis, uint32_t *frag_mask, char *ids, int64_t *id_off) {
  if (!h || !atom_off || !bond_off || !frag_off || !id_off) return DS_ERR_INVALID_ARG;
  const int64_t n = (int64_t)h->mols.size();
  atom_off[0] = bond_off[0] = frag_off[0] = 0;
  id_off[0] = 0;
  for (int64_t k = 0; k < n; ++k) {
    const LigqMol &m = h->mols[k];
    atom_off[k + 1] = atom_off[k] + (int32_t)m.type.size();
    bond_off[k + 1] = bond_off[k] + (int32_t)(m.bonds.size() / 2);
    frag_off[k + 1] = frag_off[k] + (int32_t)(m.axis.size() / 2);
    id_off[k + 1] = id_off[k] + (int64_t)m.id.size();
  }
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < n; ++k) {
    const LigqMol &m = h->mols[k];
    if (!m.type.empty()) {
      memcpy(atom_xyz + 3 * (size_t)atom_off[k], m.xyz.data(), m.xyz.size() * 4);
      memcpy(atom_type + atom_off[k], m.type.data(), m.type.size());
    }
    if (!m.bonds.empty()) memcpy(bonds + 2 * (size_t)bond_off[k], m.bonds.data(), m.bonds.size() * 4);
    if (!m.axis.empty()) {
      memcpy(frag_axis + 2 * (size_t)frag_off[k], m.axis.data(), m.axis.size() * 4);
      memcpy(frag_mask + (size_t)DS_MASK_WORDS * frag_off[k], m.mask.data(), m.mask.size() * 4);
    }
    if (!m.id.empty()) memcpy(ids + id_off[k], m.id.data(), m.id.size());
  }
  return DS_OK;
}

void ds_ligq_free(ds_ligq *h) { delete h; }

int ds_validate_ligands(int32_t n, const int32_t *atom_off, const int64_t *atom_type, const uint8_t *is_heavy,
                        const int32_t *bond_off, const int32_t *bonds, const int32_t *frag_off, const int32_t *frag_axis,
                        const int64_t *mv_off, const int64_t *mv, int32_t *codes) {
  if (n < 0 || !atom_off || !bond_off || !frag_off || !mv_off || !codes) return DS_ERR_INVALID_ARG;
#pragma omp parallel for schedule(dynamic, 256)
  for (int32_t i = 0; i < n; ++i) {
    std::string why;
    const int a0 = atom_off[i], f0 = frag_off[i];
    codes[i] = validate_arrays(atom_off[i + 1] - a0, (const long long *)atom_type + a0, is_heavy + a0,
                               bond_off[i + 1] - bond_off[i], bonds + 2 * (size_t)bond_off[i], frag_off[i + 1] - f0,
                               frag_axis + 2 * (size_t)f0, mv_off + f0, (const long long *)mv, &why);
  }
  return DS_OK;
}

}  // extern "C"
