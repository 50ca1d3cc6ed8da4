/*
 * gen_oracle.c — CPU ORACLE input makers (test infrastructure only; never on the product path).
 *
 * A plain C restatement of the reference's `io` generators: generate_dataset
 * (chain ligands with an exact heavy-atom count and F rotatable bonds, 1-2 H per heavy atom, capped
 * at 160 atoms, self-avoiding 1.5 Å steps; InfeasibleShape if F >= heavy - 1), the mixed-shape
 * datasets of BASELINE configs 3 / 5, the synthetic pocket atoms, build_pocket (SPEC.md:453-461,
 * g(d) of DESIGN.md §3 P18) and the seeded default InteractionTable.  The PRNG is the
 * counter-based SplitMix64 keyed by (seed, stream, global index) that DESIGN.md §3 pins, so every
 * shard of a screen is generated independently.  Only IEEE +, -, *, /, sqrt are used; built with
 * -ffp-contract=off like dock_oracle.c.
 *
 * Why it exists: bench.py's reference arm (`--impl reference`) times the CPU oracle on the box's
 * host cores and must not load the product library (libdockscreen.so) even for its inputs.  The
 * product's own generators (csrc/ds_host.cpp, csrc/ds_generate.cu) must produce the same bytes:
 * tests/test_oracle_generators.py checks that, array for array.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define GO_MAX_ATOMS 160
#define GO_MASK_WORDS 5
#define GO_N_TYPES 16

static const uint64_t kGolden = 0x9E3779B97F4A7C15ull;
enum { S_SHAPE = 1, S_HYDRO = 2, S_GEOM = 3, S_FRAG = 4, S_POCKET = 5, S_TABLE = 6 };

static uint64_t go_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

typedef struct { uint64_t x; } go_rng;

static go_rng rng_make(uint64_t seed, uint64_t stream, uint64_t index) {
  go_rng r;
  r.x = go_mix64(seed * kGolden ^ go_mix64(stream + 0x632BE59BD9B4E019ull)) + index * 0xD1B54A32D192ED03ull;
  return r;
}
static uint64_t rng_next(go_rng *r) {
  r->x += kGolden;
  return go_mix64(r->x);
}
static double rng_u01(go_rng *r) { return (double)(rng_next(r) >> 11) * (1.0 / 9007199254740992.0); }
static uint32_t rng_below(go_rng *r, uint32_t n) { return (uint32_t)((rng_next(r) >> 32) % n); }
/* rejection-sampled unit vector */
static void rng_unit(go_rng *r, double v[3]) {
  for (;;) {
    double x = 2.0 * rng_u01(r) - 1.0, y = 2.0 * rng_u01(r) - 1.0, z = 2.0 * rng_u01(r) - 1.0;
    double r2 = x * x + y * y + z * z;
    if (r2 > 1e-6 && r2 <= 1.0) {
      double n = sqrt(r2);
      v[0] = x / n;
      v[1] = y / n;
      v[2] = z / n;
      return;
    }
  }
}

static double d2(const double *a, const double *b) {
  double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return dx * dx + dy * dy + dz * dz;
}

/* 1-2 hydrogens per heavy atom, total capped at 160 atoms */
static int hydrogens(int64_t seed, int64_t gi, int heavy, int *nh) {
  go_rng r = rng_make((uint64_t)seed, S_HYDRO, (uint64_t)gi);
  int total = heavy;
  for (int k = 0; k < heavy; ++k) {
    int want = 1 + (int)(rng_next(&r) & 1);
    int room = GO_MAX_ATOMS - total;
    int h = want < room ? want : room;
    if (h < 0) h = 0;
    if (nh) nh[k] = h;
    total += h;
  }
  return total;
}

/* id of generated ligand `index`: "lig_<seed>_<index>" */
int go_generated_id(int64_t seed, int64_t index, char *buf, size_t cap) {
  return snprintf(buf, cap, "lig_%lld_%lld", (long long)seed, (long long)index);
}

/* heavy ~ U{heavy_min..heavy_max}, frags ~ U{0..min(frag_max, heavy-2)} per global index */
int go_mixed_shapes(int64_t seed, int64_t first, int32_t count, int32_t hmin, int32_t hmax, int32_t fmax,
                    int32_t *shapes) {
  if (count < 0 || !shapes || hmin < 1 || hmax < hmin || hmax > GO_MAX_ATOMS || fmax < 0) return -1;
  for (int32_t i = 0; i < count; ++i) {
    go_rng r = rng_make((uint64_t)seed, S_SHAPE, (uint64_t)(first + i));
    int heavy = hmin + (int)rng_below(&r, (uint32_t)(hmax - hmin + 1));
    int cap = heavy - 2 > 0 ? heavy - 2 : 0;
    if (fmax < cap) cap = fmax;
    shapes[2 * i] = heavy;
    shapes[2 * i + 1] = (int)rng_below(&r, (uint32_t)(cap + 1));
  }
  return 0;
}

static int cmp_int(const void *a, const void *b) { return *(const int *)a - *(const int *)b; }

/* SPEC.md:443 generate_dataset for ligands first .. first+count-1 with the given shapes.
 * Pass 1 (xyz == NULL) fills the CSR offsets; pass 2 the payload.  Returns -7 (InfeasibleShape). */
int go_generate_ligands(int64_t seed, int64_t first, int32_t count, const int32_t *shapes, int32_t *atom_off,
                        int32_t *frag_off, float *xyz, uint8_t *type, int32_t *frag_axis, uint32_t *frag_mask) {
  for (int32_t i = 0; i < count; ++i) {
    int heavy = shapes[2 * i], frags = shapes[2 * i + 1];
    if (heavy < 1 || heavy > GO_MAX_ATOMS || frags < 0 || (frags > 0 && frags >= heavy - 1)) return -7;
  }
  if (!xyz) {
    atom_off[0] = frag_off[0] = 0;
    for (int32_t i = 0; i < count; ++i) {
      atom_off[i + 1] = atom_off[i] + hydrogens(seed, first + i, shapes[2 * i], NULL);
      frag_off[i + 1] = frag_off[i] + shapes[2 * i + 1];
    }
    return 0;
  }
#pragma omp parallel for schedule(dynamic, 64)
  for (int32_t i = 0; i < count; ++i) {
    const int64_t gi = first + i;
    const int heavy = shapes[2 * i], frags = shapes[2 * i + 1];
    int nh[GO_MAX_ATOMS], parent[GO_MAX_ATOMS];
    double pos[GO_MAX_ATOMS][3];
    const int total = hydrogens(seed, gi, heavy, nh);
    go_rng g = rng_make((uint64_t)seed, S_GEOM, (uint64_t)gi);
    pos[0][0] = pos[0][1] = pos[0][2] = 0.0;
    parent[0] = -1;
    for (int k = 1; k < heavy; ++k) { /* self-avoiding chain: >= 1.4 Å from earlier non-neighbours */
      double cand[3];
      for (int attempt = 0; attempt < 64; ++attempt) {
        double u[3];
        rng_unit(&g, u);
        for (int c = 0; c < 3; ++c) cand[c] = pos[k - 1][c] + 1.5 * u[c];
        int ok = 1;
        for (int j = 0; j + 1 < k && ok; ++j) ok = d2(cand, pos[j]) >= 1.4 * 1.4;
        if (ok) break;
      }
      for (int c = 0; c < 3; ++c) pos[k][c] = cand[c];
      parent[k] = k - 1;
    }
    int a = heavy;
    for (int k = 0; k < heavy; ++k) /* hydrogens at 1.0 Å, >= 0.9 Å from other atoms if possible */
      for (int h = 0; h < nh[k]; ++h, ++a) {
        double cand[3];
        for (int attempt = 0; attempt < 16; ++attempt) {
          double u[3];
          rng_unit(&g, u);
          for (int c = 0; c < 3; ++c) cand[c] = pos[k][c] + 1.0 * u[c];
          int ok = 1;
          for (int j = 0; j < a && ok; ++j)
            if (j != k) ok = d2(cand, pos[j]) >= 0.9 * 0.9;
          if (ok) break;
        }
        for (int c = 0; c < 3; ++c) pos[a][c] = cand[c];
        parent[a] = k;
      }
    const int ao = atom_off[i];
    for (int k = 0; k < total; ++k) {
      for (int c = 0; c < 3; ++c) xyz[3 * (ao + k) + c] = (float)pos[k][c];
      type[ao + k] = k < heavy ? (uint8_t)(1 + rng_below(&g, GO_N_TYPES - 1)) : (uint8_t)0;
    }
    /* F distinct chain bonds (k, k+1), k in [0, heavy-3], ascending; moving side = tail minus axis_end */
    go_rng fr = rng_make((uint64_t)seed, S_FRAG, (uint64_t)gi);
    int cb[GO_MAX_ATOMS];
    const int nb = heavy - 2;
    for (int k = 0; k < nb; ++k) cb[k] = k;
    for (int f = 0; f < frags; ++f) {
      int j = f + (int)rng_below(&fr, (uint32_t)(nb - f));
      int t = cb[f];
      cb[f] = cb[j];
      cb[j] = t;
    }
    qsort(cb, (size_t)frags, sizeof(int), cmp_int);
    const int fo = frag_off[i];
    for (int f = 0; f < frags; ++f) {
      const int k = cb[f];
      frag_axis[2 * (fo + f)] = k;
      frag_axis[2 * (fo + f) + 1] = k + 1;
      uint32_t *m = frag_mask + (size_t)GO_MASK_WORDS * (fo + f);
      for (int w = 0; w < GO_MASK_WORDS; ++w) m[w] = 0;
      for (int t = 0; t < total; ++t) {
        const int root = t < heavy ? t : parent[t];
        if (root >= k + 1 && t != k + 1) m[t >> 5] |= 1u << (t & 31);
      }
    }
  }
  return 0;
}

/* synthetic pocket atoms: uniform in the shell rmin <= r <= rmax, types 1..15 */
int go_pocket_atoms(int64_t seed, int32_t n, float rmin, float rmax, float *xyz, uint8_t *type) {
  go_rng r = rng_make((uint64_t)seed, S_POCKET, 0);
  const double lo2 = (double)rmin * rmin, hi2 = (double)rmax * rmax;
  for (int32_t i = 0; i < n; ++i) {
    double p[3];
    for (;;) {
      for (int c = 0; c < 3; ++c) p[c] = (2.0 * rng_u01(&r) - 1.0) * (double)rmax;
      double q = p[0] * p[0] + p[1] * p[1] + p[2] * p[2];
      if (q >= lo2 && q <= hi2) break;
    }
    for (int c = 0; c < 3; ++c) xyz[3 * i + c] = (float)p[c];
    type[i] = (uint8_t)(1 + rng_below(&r, GO_N_TYPES - 1));
  }
  return 0;
}

/* SPEC.md:453 build_pocket: bounding box + padding, node = rint(10 g(d)) (P18); values NULL: sizes */
int go_build_pocket(const float *xyz, int32_t n, float spacing, float padding, float origin[3], int32_t dims[3],
                    int32_t *values) {
  if (n <= 0) return -6;
  double lo[3], hi[3];
  for (int c = 0; c < 3; ++c) lo[c] = hi[c] = xyz[c];
  for (int i = 1; i < n; ++i)
    for (int c = 0; c < 3; ++c) {
      double v = xyz[3 * i + c];
      if (v < lo[c]) lo[c] = v;
      if (v > hi[c]) hi[c] = v;
    }
  for (int c = 0; c < 3; ++c) {
    origin[c] = (float)(lo[c] - (double)padding);
    double span = (hi[c] + (double)padding) - (double)origin[c];
    dims[c] = (int32_t)ceil(span / (double)spacing - 1e-9) + 1;
    if (dims[c] < 1) dims[c] = 1;
  }
  if (!values) return 0;
  const int nx = dims[0], ny = dims[1], nz = dims[2];
#pragma omp parallel for schedule(static) collapse(2)
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        const double node[3] = {(double)origin[0] + x * (double)spacing, (double)origin[1] + y * (double)spacing,
                                (double)origin[2] + z * (double)spacing};
        double best = INFINITY;
        for (int i = 0; i < n; ++i) {
          const double a[3] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
          double q = d2(node, a);
          if (q < best) best = q;
        }
        const double d = sqrt(best);
        double g;
        if (d <= 3.0) g = -1.0 + 2.0 * d / 3.0;
        else if (d <= 5.0) g = 1.0;
        else if (d <= 8.0) g = 1.0 - 2.0 * (d - 5.0) / 3.0;
        else g = -1.0;
        values[(size_t)x + (size_t)nx * ((size_t)y + (size_t)ny * z)] = (int32_t)nearbyint(10.0 * g);
      }
  return 0;
}

/* SPEC.md:221 default table: symmetric 16x16, seeded, uniform in [-1, 1] */
int go_default_table(int64_t seed, float *table) {
  go_rng r = rng_make((uint64_t)seed, S_TABLE, 0);
  for (int i = 0; i < GO_N_TYPES; ++i)
    for (int j = i; j < GO_N_TYPES; ++j) {
      float w = (float)(2.0 * rng_u01(&r) - 1.0);
      table[i * GO_N_TYPES + j] = table[j * GO_N_TYPES + i] = w;
    }
  return 0;
}
