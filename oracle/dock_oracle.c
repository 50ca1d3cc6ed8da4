/*
 * dock_oracle.c — CPU ORACLE (test infrastructure only; never on the product path).
 *
 * A plain, sequential C restatement of the reference docking pipeline: SPEC.md's `docking`
 * module (Alg. 1 of PAPER.md:208-252) over the `transform` and `scoring` L2 kernels that the
 * reference places in its native slot `dockscreen.kernels._core` (pkg/setup.py:10-18; source
 * absent from the reference).  Built like that slot: -O3, IEEE-exact, no fast-math and no FMA
 * contraction (pkg/setup.py:5-6, 16) — every fused multiply-add below is an explicit fmaf().
 *
 * Parity status: the reference ships no code, tests or golden vectors.
 * This oracle is pinned to the SPEC's known-answer examples (tests/test_oracle_kat.py) and
 * cross-checked against an independent exact-arithmetic Python restatement
 * (oracle/pyoracle.py, tests/test_oracle_crosscheck.py).  The numeric recipe it follows is
 * DESIGN.md §3 (pins P0-P18); the pins are ours because the SPEC leaves them open.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may load this file.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAX_ATOMS 160
#define OR_MASK_WORDS 5
#define OR_N_TYPES 16
#define OR_MAX_BINS 8
#define OR_MAX_RESTARTS 32
#define OR_OUTSIDE (-100)

/* ---------------------------------------------------------------- inputs / outputs */
typedef struct {
  float origin[3];
  float spacing;
  int32_t dims[3];
  const int32_t *values;   /* x-fastest */
  int32_t n_atoms;
  const float *atom_xyz;   /* Å */
  const uint8_t *atom_type;
  const float *table;      /* 16x16 */
  int32_t n_bins;
  const float *bin_ub;
  const float *bin_mult;
} or_pocket;

typedef struct {
  int32_t restarts_n, rescore_top_k, alignment_step_deg, torsion_step_deg;
  float bump_distance, similarity_rmsd, rescore_cutoff;
  int32_t early_exit;
  int64_t seed;
} or_config;

typedef struct {
  int32_t status;          /* 0 ok, 1 no valid pose, 2 degenerate axis */
  int32_t geom_score;
  int64_t chem_fx;
  int32_t best_restart, best_ax, best_ay, n_kept;
  int64_t poses_scored;
  int64_t bump_checks;     /* sequential pair evaluations */
  int64_t bump_checks_rows; /* the same scan counted in whole moving-atom rows (device granularity, P14) */
  int64_t bump_early_exits;
} or_result;

typedef struct {
  int32_t align_score, final_geom, ax, ay, valid, kept;
} or_restart;

/* ---------------------------------------------------------------- P0: trig table */
static float g_cos[360], g_sin[360];
static int g_trig_ready = 0;
static void trig_init(void) {
  if (g_trig_ready) return;
  for (int d = 0; d < 360; ++d) {
    double rad = (double)d * 0.017453292519943295;
    g_cos[d] = (float)cos(rad);
    g_sin[d] = (float)sin(rad);
  }
  g_trig_ready = 1;
}

/* SPEC.md:117-133 rot_x / rot_y (right-handed, active), plus rot_z for the start pose */
static void rot_x(int deg, float m[9]) {
  float c = g_cos[deg], s = g_sin[deg];
  float r[9] = {1.f, 0.f, 0.f, 0.f, c, -s, 0.f, s, c};
  memcpy(m, r, sizeof r);
}
static void rot_y(int deg, float m[9]) {
  float c = g_cos[deg], s = g_sin[deg];
  float r[9] = {c, 0.f, s, 0.f, 1.f, 0.f, -s, 0.f, c};
  memcpy(m, r, sizeof r);
}
static void rot_z(int deg, float m[9]) {
  float c = g_cos[deg], s = g_sin[deg];
  float r[9] = {c, -s, 0.f, s, c, 0.f, 0.f, 0.f, 1.f};
  memcpy(m, r, sizeof r);
}

/* P1: C = A (x) B, C_ij = fma(A_i2, B_2j, fma(A_i1, B_1j, A_i0 * B_0j)) */
static void mat3_mul(const float *A, const float *B, float *C) {
  float t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      t[3 * i + j] = fmaf(A[3 * i + 2], B[6 + j], fmaf(A[3 * i + 1], B[3 + j], A[3 * i] * B[j]));
  memcpy(C, t, sizeof t);
}

/* ---------------------------------------------------------------- P5: PRNG */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t or_fnv1a64(const char *s, size_t n) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= (unsigned char)s[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

/* ---------------------------------------------------------------- pocket in grid frame */
typedef struct {
  const or_pocket *p;
  float inv_s;
  float patom[4 * 4096]; /* grid-frame pocket atoms (x, y, z) + type, up to 4096 atoms */
  int32_t *wfx;          /* [16][16][nb+1] */
  float ub2[OR_MAX_BINS];
  int nb;
} or_pk;

static int pk_init(or_pk *k, const or_pocket *p) {
  k->p = p;
  k->inv_s = (float)(1.0 / (double)p->spacing);
  if (p->n_atoms > 4096) return -1;
  for (int j = 0; j < p->n_atoms; ++j) {
    for (int c = 0; c < 3; ++c)
      k->patom[4 * j + c] = (float)(((double)p->atom_xyz[3 * j + c] - (double)p->origin[c]) / (double)p->spacing);
    k->patom[4 * j + 3] = (float)p->atom_type[j];
  }
  k->nb = p->n_bins;
  for (int b = 0; b < p->n_bins; ++b) {
    double ub = (double)p->bin_ub[b] / (double)p->spacing;
    k->ub2[b] = (float)(ub * ub);
  }
  k->wfx = (int32_t *)calloc((size_t)OR_N_TYPES * OR_N_TYPES * (p->n_bins + 1), sizeof(int32_t));
  for (int t = 0; t < OR_N_TYPES * OR_N_TYPES; ++t)
    for (int b = 0; b < p->n_bins; ++b) {
      float prod = p->table[t] * p->bin_mult[b];
      k->wfx[t * (p->n_bins + 1) + b] = (int32_t)llrint((double)prod * 16777216.0);
    }
  return 0;
}
static void pk_free(or_pk *k) { free(k->wfx); }

/* ---------------------------------------------------------------- SPEC.md:183 grid_score (grid frame) */
static int grid_value(const or_pk *k, const float u[3]) {
  const or_pocket *p = k->p;
  float n[3];
  for (int c = 0; c < 3; ++c) {
    n[c] = rintf(u[c]);  /* P4: nearest node, ties to even */
    if (!(n[c] >= 0.0f && n[c] <= (float)(p->dims[c] - 1))) return OR_OUTSIDE;
  }
  long ix = (long)n[0], iy = (long)n[1], iz = (long)n[2];
  return p->values[ix + (long)p->dims[0] * (iy + (long)p->dims[1] * iz)];
}
static int grid_score(const or_pk *k, const float (*u)[3], int n) {
  int s = 0;
  for (int i = 0; i < n; ++i) s += grid_value(k, u[i]);
  return s;
}

/* ---------------------------------------------------------------- ligand */
typedef struct {
  int A, F, H;
  float d[OR_MAX_ATOMS][3]; /* centred coordinates (P2) */
  uint8_t type[OR_MAX_ATOMS];
  const int32_t *axis;      /* 2 per fragment */
  const uint32_t *mask;     /* 5 words per fragment */
  uint64_t idh;
} or_lig;

static int in_mask(const uint32_t *m, int i) { return (m[i >> 5] >> (i & 31)) & 1; }

/* SPEC.md:237 generate_starting_pose -> R0s (rotation scaled to the grid frame) and t (grid frame) */
static void starting_pose(const or_lig *L, const or_pk *k, int r, int64_t seed, float R0s[9], float t[3]) {
  const uint64_t base = L->idh ^ ((uint64_t)seed * 0x9E3779B97F4A7C15ull);
  uint64_t z[6];
  for (int j = 0; j < 6; ++j) z[j] = mix64(base + (uint64_t)(r * 8 + j + 1) * 0x9E3779B97F4A7C15ull);
  for (int c = 0; c < 3; ++c) {
    float U = (float)(uint32_t)(z[c] >> 40) * 5.9604644775390625e-08f;
    float a = 0.8f * U;
    float b = 0.1f + a;
    t[c] = (float)(k->p->dims[c] - 1) * b;
  }
  float Rx[9], Ry[9], Rz[9], Ryx[9], R0[9];
  rot_x((int)((z[3] >> 32) % 360u), Rx);
  rot_y((int)((z[4] >> 32) % 360u), Ry);
  rot_z((int)((z[5] >> 32) % 360u), Rz);
  mat3_mul(Ry, Rx, Ryx);
  mat3_mul(Rz, Ryx, R0);
  for (int q = 0; q < 9; ++q) R0s[q] = R0[q] * k->inv_s;
}

/* P6: coordinates of the rigid pose (ax, ay) of a restart, x rotation first then y (Alg. 1
 * lines 4-6; apply_rigid of SPEC.md:135 about the centroid t, fresh from the starting pose,
 * SPEC.md:303): R' = Rx(ax) (x) R0s, v = R' d, u = Ry(ay) v + t written out as
 * u_x = fma(sy, v_z, fma(cy, v_x, t_x)), u_y = v_y + t_y, u_z = fma(cy, v_z, fma(-sy, v_x, t_z)). */
static void rigid_pose(const or_lig *L, const float R0s[9], const float t[3], int ax_deg, int ay_deg,
                       float (*u)[3]) {
  float Rx[9], Rp[9];
  rot_x(ax_deg, Rx);
  mat3_mul(Rx, R0s, Rp);
  const float cy = g_cos[ay_deg], sy = g_sin[ay_deg];
  for (int i = 0; i < L->A; ++i) {
    const float *d = L->d[i];
    float v[3];
    for (int k = 0; k < 3; ++k) v[k] = fmaf(Rp[3 * k + 2], d[2], fmaf(Rp[3 * k + 1], d[1], Rp[3 * k] * d[0]));
    u[i][0] = fmaf(sy, v[2], fmaf(cy, v[0], t[0]));
    u[i][1] = v[1] + t[1];
    u[i][2] = fmaf(cy, v[2], fmaf(-sy, v[0], t[2]));
  }
}

/* SPEC.md:247 align: exhaustive (ix, iy) sweep, ties -> smallest (ax, ay) */
static int align_pose(const or_lig *L, const or_pk *k, const or_config *cfg, const float R0s[9], const float t[3],
                      int *bix, int *biy, float (*u)[3]) {
  const int na = 360 / cfg->alignment_step_deg;
  int best = 0, have = 0;
  float tmp[OR_MAX_ATOMS][3];
  for (int ix = 0; ix < na; ++ix)
    for (int iy = 0; iy < na; ++iy) {
      rigid_pose(L, R0s, t, ix * cfg->alignment_step_deg, iy * cfg->alignment_step_deg, tmp);
      int s = grid_score(k, (const float(*)[3])tmp, L->A);
      if (!have || s > best) {
        best = s;
        *bix = ix;
        *biy = iy;
        have = 1;
      }
    }
  rigid_pose(L, R0s, t, *bix * cfg->alignment_step_deg, *biy * cfg->alignment_step_deg, u);
  return best;
}

/* P8: Rodrigues matrix from unit axis and table angle */
static void torsion_matrix(float kx, float ky, float kz, int deg, float R[9]) {
  float c = g_cos[deg], s = g_sin[deg];
  float C = 1.0f - c;
  float Ckx = C * kx, Cky = C * ky, Ckz = C * kz;
  float skx = s * kx, sky = s * ky, skz = s * kz;
  R[0] = fmaf(Ckx, kx, c);
  R[1] = fmaf(Ckx, ky, -skz);
  R[2] = fmaf(Ckx, kz, sky);
  R[3] = fmaf(Cky, kx, skz);
  R[4] = fmaf(Cky, ky, c);
  R[5] = fmaf(Cky, kz, -skx);
  R[6] = fmaf(Ckz, kx, -sky);
  R[7] = fmaf(Ckz, ky, skx);
  R[8] = fmaf(Ckz, kz, c);
}

/* SPEC.md:145 apply_torsion (grid frame). Returns -1 on DegenerateAxis. Angle 0 is the identity. */
static int apply_torsion(const or_lig *L, int f, const float (*u)[3], int deg, float eps, float (*out)[3]) {
  const int ab = L->axis[2 * f], ae = L->axis[2 * f + 1];
  const uint32_t *m = L->mask + OR_MASK_WORDS * f;
  memcpy(out, u, sizeof(float) * 3 * L->A);
  float vx = u[ae][0] - u[ab][0], vy = u[ae][1] - u[ab][1], vz = u[ae][2] - u[ab][2];
  float len = sqrtf(fmaf(vz, vz, fmaf(vy, vy, vx * vx)));
  if (!(len >= eps)) return -1;
  if (deg == 0) return 0;
  float kx = vx / len, ky = vy / len, kz = vz / len, R[9];
  torsion_matrix(kx, ky, kz, deg, R);
  const float *a = u[ab];
  for (int i = 0; i < L->A; ++i) {
    if (!in_mask(m, i)) continue;
    float wx = u[i][0] - a[0], wy = u[i][1] - a[1], wz = u[i][2] - a[2];
    out[i][0] = fmaf(R[2], wz, fmaf(R[1], wy, fmaf(R[0], wx, a[0])));
    out[i][1] = fmaf(R[5], wz, fmaf(R[4], wy, fmaf(R[3], wx, a[1])));
    out[i][2] = fmaf(R[8], wz, fmaf(R[7], wy, fmaf(R[6], wx, a[2])));
  }
  return 0;
}

/* SPEC.md:193 bump_check: i in mask (ascending) x j not in mask and not an axis atom (ascending) */
static int bump_check(const or_lig *L, int f, const float (*u)[3], float bd2, int early_exit, int64_t *pairs,
                      int64_t *pairs_rows, int64_t *exits) {
  const int ab = L->axis[2 * f], ae = L->axis[2 * f + 1];
  const uint32_t *m = L->mask + OR_MASK_WORDS * f;
  int64_t n = 0, total = 0, rows = 0;
  int bump = 0, nm = 0, nc = 0;
  for (int i = 0; i < L->A; ++i) {
    if (in_mask(m, i)) ++nm;
    else if (i != ab && i != ae) ++nc;
  }
  total = (int64_t)nm * nc;
  for (int i = 0; i < L->A && !(bump && early_exit); ++i) {
    if (!in_mask(m, i)) continue;
    rows += nc;
    for (int j = 0; j < L->A; ++j) {
      if (in_mask(m, j) || j == ab || j == ae) continue;
      float dx = u[i][0] - u[j][0], dy = u[i][1] - u[j][1], dz = u[i][2] - u[j][2];
      float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      ++n;
      if (d2 < bd2) {
        bump = 1;
        if (early_exit) break;
      }
    }
  }
  *pairs += n;
  *pairs_rows += early_exit && bump ? rows : total;
  if (bump && early_exit) ++*exits;
  return bump;
}

/* ---------------------------------------------------------------- SPEC.md:277 dock_ligand */
/* One restart of Alg. 1 (starting pose, align, optimize_pose) into U; its own counters in *cnt.
 * Returns 2 on DegenerateAxis (cnt then holds the counts up to that point, like the sequential
 * scan), else 0. */
typedef struct {
  int64_t poses_scored, bump_checks, bump_checks_rows, bump_early_exits;
  int geom, valid, ax, ay, align_score;
} or_restart_out;

static int dock_restart(const or_lig *L, const or_pk *k, const or_config *cfg, int r, float (*U)[3],
                        uint8_t *tors /* F*N or NULL */, or_restart_out *o) {
  const int N = cfg->restarts_n, na = 360 / cfg->alignment_step_deg, nt = 360 / cfg->torsion_step_deg;
  const double s = (double)k->p->spacing;
  const float bd2 = (float)(((double)cfg->bump_distance / s) * ((double)cfg->bump_distance / s));
  const float eps = (float)(1e-9 / s);
  memset(o, 0, sizeof *o);
  float R0s[9], t[3];
  starting_pose(L, k, r, cfg->seed, R0s, t);
  int ix = 0, iy = 0;
  o->align_score = align_pose(L, k, cfg, R0s, t, &ix, &iy, U);
  o->poses_scored += (int64_t)na * na;
  o->ax = ix;
  o->ay = iy;
  /* SPEC.md:257 optimize_pose */
  int all_bumped = 0;
  for (int f = 0; f < L->F; ++f) {
    float cand[OR_MAX_ATOMS][3];
    int best = 0, best_k = -1;
    for (int a = 0; a < nt; ++a) {
      if (apply_torsion(L, f, (const float(*)[3])U, a * cfg->torsion_step_deg, eps, cand) < 0 && nt > 1)
        return 2; /* DegenerateAxis */
      o->poses_scored += 1;
      if (bump_check(L, f, (const float(*)[3])cand, bd2, cfg->early_exit, &o->bump_checks, &o->bump_checks_rows,
                     &o->bump_early_exits))
        continue;
      int sc = grid_score(k, (const float(*)[3])cand, L->A);
      if (best_k < 0 || sc > best) {
        best = sc;
        best_k = a;
      }
    }
    if (best_k > 0) {
      apply_torsion(L, f, (const float(*)[3])U, best_k * cfg->torsion_step_deg, eps, cand);
      memcpy(U, cand, sizeof(float) * 3 * L->A);
    }
    if (best_k < 0) ++all_bumped;
    if (tors) tors[f * N + r] = best_k < 0 ? 255 : (uint8_t)best_k;
  }
  o->valid = !(L->F >= 1 && all_bumped == L->F);
  o->geom = grid_score(k, (const float(*)[3])U, L->A);
  return 0;
}

/* dock_ligand; inner_threads > 1 runs the restarts on an inner pool (the latency engine's
 * pose-level parallelism) with results identical to the sequential loop. */
static int dock_ligand_impl(const or_lig *L, const or_pk *k, const or_config *cfg, or_result *res, or_restart *rr,
                            uint8_t *tors, float *best_xyz, int inner_threads, float *restart_xyz) {
  trig_init();
  const int N = cfg->restarts_n;
  const double thr = (double)cfg->similarity_rmsd / (double)k->p->spacing;
  const double thr2 = thr * thr;
  static __thread float U[OR_MAX_RESTARTS][OR_MAX_ATOMS][3];
  or_restart_out ro[OR_MAX_RESTARTS];
  int st[OR_MAX_RESTARTS];
  int geom[OR_MAX_RESTARTS], valid[OR_MAX_RESTARTS], aix[OR_MAX_RESTARTS], aiy[OR_MAX_RESTARTS];
  memset(res, 0, sizeof *res);
  float(*Ub)[OR_MAX_ATOMS][3] = U; /* the calling thread's buffer, shared with the inner pool */
  if (inner_threads > 1) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(inner_threads)
    for (int r = 0; r < N; ++r) st[r] = dock_restart(L, k, cfg, r, Ub[r], tors, &ro[r]);
  } else {
    for (int r = 0; r < N; ++r)
      if ((st[r] = dock_restart(L, k, cfg, r, Ub[r], tors, &ro[r])) != 0) {
        for (int q = r + 1; q < N; ++q) st[q] = -1;
        break;
      }
  }
  for (int r = 0; r < N; ++r) {
    res->poses_scored += ro[r].poses_scored;
    res->bump_checks += ro[r].bump_checks;
    res->bump_checks_rows += ro[r].bump_checks_rows;
    res->bump_early_exits += ro[r].bump_early_exits;
    if (st[r] == 2) { /* the sequential loop stops here: later restarts never ran */
      res->status = 2;
      if (tors)
        for (int q = r + 1; q < N; ++q)
          for (int f = 0; f < L->F; ++f) tors[f * N + q] = 0;
      return 2;
    }
    geom[r] = ro[r].geom;
    valid[r] = ro[r].valid;
    aix[r] = ro[r].ax;
    aiy[r] = ro[r].ay;
    if (rr) {
      rr[r].align_score = ro[r].align_score;
      rr[r].final_geom = geom[r];
      rr[r].ax = aix[r];
      rr[r].ay = aiy[r];
      rr[r].valid = valid[r];
      rr[r].kept = 0;
    }
  }
  float(*Uc)[OR_MAX_ATOMS][3] = Ub;
#define U Uc
  /* SPEC.md:267 select_poses: valid poses by (geom desc, restart asc), greedy heavy-atom RMSD >= thr */
  int ord[OR_MAX_RESTARTS], nv = 0;
  for (int r = 0; r < N; ++r)
    if (valid[r]) ord[nv++] = r;
  if (nv == 0) {
    res->status = 1; /* NoValidPose */
    return 1;
  }
  for (int a = 1; a < nv; ++a) /* insertion sort: stable on restart order */
    for (int b = a; b > 0 && geom[ord[b]] > geom[ord[b - 1]]; --b) {
      int tmp = ord[b];
      ord[b] = ord[b - 1];
      ord[b - 1] = tmp;
    }
  int kept[OR_MAX_RESTARTS], nk = 0;
  for (int o = 0; o < nv && nk < cfg->rescore_top_k; ++o) {
    int c = ord[o], ok = 1;
    for (int q = 0; q < nk && ok; ++q) {
      double sum = 0.0;
      for (int i = 0; i < L->A; ++i) {
        if (L->type[i] == 0) continue;
        double dx = (double)U[c][i][0] - (double)U[kept[q]][i][0];
        double dy = (double)U[c][i][1] - (double)U[kept[q]][i][1];
        double dz = (double)U[c][i][2] - (double)U[kept[q]][i][2];
        double tt = dx * dx;
        tt = tt + dy * dy;
        tt = tt + dz * dz;
        sum = sum + tt;
      }
      ok = L->H > 0 && sum >= thr2 * (double)L->H;
    }
    if (ok) kept[nk++] = c;
  }
  /* SPEC.md:203 rescore (fixed point, exact) and best = max chem, ties -> restart asc */
  int64_t best_chem = 0;
  int best_r = -1;
  for (int q = 0; q < nk; ++q) {
    int r = kept[q];
    int64_t acc = 0;
    for (int i = 0; i < L->A; ++i)
      for (int j = 0; j < k->p->n_atoms; ++j) {
        const float *y = k->patom + 4 * j;
        float dx = U[r][i][0] - y[0], dy = U[r][i][1] - y[1], dz = U[r][i][2] - y[2];
        float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        int b = 0;
        for (int qq = 0; qq < k->nb; ++qq) b += !(d2 < k->ub2[qq]);
        acc += k->wfx[((int)L->type[i] * OR_N_TYPES + (int)y[3]) * (k->nb + 1) + b];
      }
    if (best_r < 0 || acc > best_chem || (acc == best_chem && r < best_r)) {
      best_chem = acc;
      best_r = r;
    }
    if (rr) rr[r].kept = q + 1;
  }
  res->status = 0;
  res->geom_score = geom[best_r];
  res->chem_fx = best_chem;
  res->best_restart = best_r;
  res->best_ax = aix[best_r];
  res->best_ay = aiy[best_r];
  res->n_kept = nk;
  if (best_xyz)
    for (int i = 0; i < L->A; ++i)
      for (int c = 0; c < 3; ++c) best_xyz[3 * i + c] = fmaf(U[best_r][i][c], k->p->spacing, k->p->origin[c]);
  if (restart_xyz) /* every restart's final pose in Å (N x A x 3), for tests of the rescore semantics */
    for (int r = 0; r < N; ++r)
      for (int i = 0; i < L->A; ++i)
        for (int c = 0; c < 3; ++c)
          restart_xyz[3 * ((size_t)r * L->A + i) + c] = fmaf(U[r][i][c], k->p->spacing, k->p->origin[c]);
  return 0;
#undef U
}

int or_dock_ligand(const or_lig *L, const or_pk *k, const or_config *cfg, or_result *res, or_restart *rr,
                   uint8_t *tors /* F*N: [f*N + r] */, float *best_xyz /* A*3 Å, may be NULL */) {
  return dock_ligand_impl(L, k, cfg, res, rr, tors, best_xyz, 1, NULL);
}

/* P2: c0 = f32(f64 sequential mean), d = f32(p - c0) */
static void lig_init(or_lig *L, int A, const float *xyz, const uint8_t *type, int F, const int32_t *axis,
                     const uint32_t *mask, const char *id, size_t idlen) {
  L->A = A;
  L->F = F;
  L->axis = axis;
  L->mask = mask;
  L->H = 0;
  double sm[3] = {0, 0, 0};
  for (int i = 0; i < A; ++i)
    for (int c = 0; c < 3; ++c) sm[c] += (double)xyz[3 * i + c];
  float c0[3];
  for (int c = 0; c < 3; ++c) c0[c] = (float)(sm[c] / (double)A);
  for (int i = 0; i < A; ++i) {
    for (int c = 0; c < 3; ++c) L->d[i][c] = xyz[3 * i + c] - c0[c];
    L->type[i] = type[i];
    L->H += type[i] != 0;
  }
  L->idh = or_fnv1a64(id, idlen);
}

/* Batch entry (ctypes).  CSR inputs as produced by the generators; OpenMP over ligands is the
 * SPEC's batched CPU engine shape ("one sequential worker per ligand"). */
int or_dock_batch(int n, const int32_t *atom_off, const float *atom_xyz, const uint8_t *atom_type,
                  const int32_t *frag_off, const int32_t *frag_axis, const uint32_t *frag_mask, const char *ids,
                  const int64_t *id_off, const or_pocket *pocket, const or_config *cfg, int threads,
                  or_result *res, or_restart *rr /* n*N, may be NULL */, uint8_t *tors /* frag_off[n]*N */,
                  float *best_xyz /* atom_off[n]*3, may be NULL */) {
  trig_init();
  or_pk *k = (or_pk *)malloc(sizeof(or_pk));
  if (pk_init(k, pocket)) {
    free(k);
    return -1;
  }
  const int N = cfg->restarts_n;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : 1)
  for (int i = 0; i < n; ++i) {
    or_lig L;
    lig_init(&L, atom_off[i + 1] - atom_off[i], atom_xyz + 3 * (size_t)atom_off[i], atom_type + atom_off[i],
             frag_off[i + 1] - frag_off[i], frag_axis + 2 * (size_t)frag_off[i],
             frag_mask + (size_t)OR_MASK_WORDS * frag_off[i], ids + id_off[i], (size_t)(id_off[i + 1] - id_off[i]));
    or_dock_ligand(&L, k, cfg, res + i, rr ? rr + (size_t)i * N : NULL, tors ? tors + (size_t)frag_off[i] * N : NULL,
                   best_xyz ? best_xyz + 3 * (size_t)atom_off[i] : NULL);
  }
  pk_free(k);
  free(k);
  return 0;
}

/* The latency engine's CPU shape: ligands one after another, each ligand's
 * restarts spread over an inner pool of `threads` workers; results identical to or_dock_batch. */
int or_dock_batch_latency(int n, const int32_t *atom_off, const float *atom_xyz, const uint8_t *atom_type,
                          const int32_t *frag_off, const int32_t *frag_axis, const uint32_t *frag_mask,
                          const char *ids, const int64_t *id_off, const or_pocket *pocket, const or_config *cfg,
                          int threads, or_result *res, or_restart *rr, uint8_t *tors, float *best_xyz) {
  trig_init();
  or_pk *k = (or_pk *)malloc(sizeof(or_pk));
  if (pk_init(k, pocket)) {
    free(k);
    return -1;
  }
  const int N = cfg->restarts_n;
  for (int i = 0; i < n; ++i) {
    or_lig L;
    lig_init(&L, atom_off[i + 1] - atom_off[i], atom_xyz + 3 * (size_t)atom_off[i], atom_type + atom_off[i],
             frag_off[i + 1] - frag_off[i], frag_axis + 2 * (size_t)frag_off[i],
             frag_mask + (size_t)OR_MASK_WORDS * frag_off[i], ids + id_off[i], (size_t)(id_off[i + 1] - id_off[i]));
    dock_ligand_impl(&L, k, cfg, res + i, rr ? rr + (size_t)i * N : NULL, tors ? tors + (size_t)frag_off[i] * N : NULL,
                     best_xyz ? best_xyz + 3 * (size_t)atom_off[i] : NULL, threads > 1 ? threads : 1, NULL);
  }
  pk_free(k);
  free(k);
  return 0;
}

/* ---------------------------------------------------------------- L2 ops in Å (SPEC examples) */
static void to_grid_frame(const or_pk *k, const float q[3], float u[3]) {
  for (int c = 0; c < 3; ++c) {
    float off = (float)(-(double)k->p->origin[c] / (double)k->p->spacing);
    u[c] = fmaf(q[c], k->inv_s, off);
  }
}
int or_grid_score(const or_pocket *p, const float *coords, int n) {
  or_pk *k = (or_pk *)malloc(sizeof(or_pk));
  pk_init(k, p);
  int s = 0;
  for (int i = 0; i < n; ++i) {
    float u[3];
    to_grid_frame(k, coords + 3 * i, u);
    s += grid_value(k, u);
  }
  pk_free(k);
  free(k);
  return s;
}
int64_t or_rescore(const or_pocket *p, const float *coords, const uint8_t *types, int n) {
  or_pk *k = (or_pk *)malloc(sizeof(or_pk));
  pk_init(k, p);
  int64_t acc = 0;
  for (int i = 0; i < n; ++i) {
    float u[3];
    to_grid_frame(k, coords + 3 * i, u);
    for (int j = 0; j < p->n_atoms; ++j) {
      const float *y = k->patom + 4 * j;
      float dx = u[0] - y[0], dy = u[1] - y[1], dz = u[2] - y[2];
      float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
      int b = 0;
      for (int qq = 0; qq < k->nb; ++qq) b += !(d2 < k->ub2[qq]);
      acc += k->wfx[((int)types[i] * OR_N_TYPES + (int)y[3]) * (k->nb + 1) + b];
    }
  }
  pk_free(k);
  free(k);
  return acc;
}
void or_rot(int axis, int deg, float *m) {
  trig_init();
  if (axis == 0) rot_x(((deg % 360) + 360) % 360, m);
  else if (axis == 1) rot_y(((deg % 360) + 360) % 360, m);
  else rot_z(((deg % 360) + 360) % 360, m);
}

/* ---------------------------------------------------------------- the other L2 ops of the native
 * slot in Å, pinned like the docking recipe: each pose of n atoms is 3n floats. */
/* SPEC.md:135 apply_rigid: p' = m (p - c) + c, w = p - c, p'_i = fma(m_i2, w_z, fma(m_i1, w_y, fma(m_i0, w_x, c_i))) */
void or_apply_rigid(int n_atoms, int n_poses, const float *coords, const float *m /* 9 per pose */,
                    const float *center /* 3 per pose */, float *out) {
  for (int p = 0; p < n_poses; ++p) {
    const float *M = m + 9 * p, *c = center + 3 * p;
    for (int i = 0; i < n_atoms; ++i) {
      const float *q = coords + 3 * ((size_t)p * n_atoms + i);
      float *o = out + 3 * ((size_t)p * n_atoms + i);
      float wx = q[0] - c[0], wy = q[1] - c[1], wz = q[2] - c[2];
      o[0] = fmaf(M[2], wz, fmaf(M[1], wy, fmaf(M[0], wx, c[0])));
      o[1] = fmaf(M[5], wz, fmaf(M[4], wy, fmaf(M[3], wx, c[1])));
      o[2] = fmaf(M[8], wz, fmaf(M[7], wy, fmaf(M[6], wx, c[2])));
    }
  }
}

/* SPEC.md:145 apply_torsion in Å (P8 with eps = f32(1e-9 Å)); status[p] = 0 or 2 (DegenerateAxis,
 * pose left unchanged) */
void or_apply_torsion(int n_atoms, int n_poses, const float *coords, int ab, int ae, const uint32_t mask[5],
                      int deg, float *out, int32_t *status) {
  trig_init();
  deg = ((deg % 360) + 360) % 360;
  for (int p = 0; p < n_poses; ++p) {
    const float(*u)[3] = (const float(*)[3])(coords + 3 * (size_t)p * n_atoms);
    float(*o)[3] = (float(*)[3])(out + 3 * (size_t)p * n_atoms);
    memcpy(o, u, sizeof(float) * 3 * n_atoms);
    float vx = u[ae][0] - u[ab][0], vy = u[ae][1] - u[ab][1], vz = u[ae][2] - u[ab][2];
    float len = sqrtf(fmaf(vz, vz, fmaf(vy, vy, vx * vx)));
    status[p] = !(len >= 1e-9f) ? 2 : 0;
    if (status[p] || deg == 0) continue;
    float R[9];
    torsion_matrix(vx / len, vy / len, vz / len, deg, R);
    const float *a = u[ab];
    for (int i = 0; i < n_atoms; ++i) {
      if (!in_mask(mask, i)) continue;
      float wx = u[i][0] - a[0], wy = u[i][1] - a[1], wz = u[i][2] - a[2];
      o[i][0] = fmaf(R[2], wz, fmaf(R[1], wy, fmaf(R[0], wx, a[0])));
      o[i][1] = fmaf(R[5], wz, fmaf(R[4], wy, fmaf(R[3], wx, a[1])));
      o[i][2] = fmaf(R[8], wz, fmaf(R[7], wy, fmaf(R[6], wx, a[2])));
    }
  }
}

/* SPEC.md:193 bump_check in Å: bd2 = f32(bump_distance^2 in f64); pairs[p] = pair evaluations of
 * the sequential scan (i in mask ascending x j in the complement minus the axis atoms ascending) */
void or_bump_check(int n_atoms, int n_poses, const float *coords, int ab, int ae, const uint32_t mask[5],
                   float bump_distance, int early_exit, uint8_t *bump, int64_t *pairs) {
  const float bd2 = (float)((double)bump_distance * (double)bump_distance);
  for (int p = 0; p < n_poses; ++p) {
    const float(*u)[3] = (const float(*)[3])(coords + 3 * (size_t)p * n_atoms);
    int64_t n = 0;
    int hit = 0;
    for (int i = 0; i < n_atoms && !(hit && early_exit); ++i) {
      if (!in_mask(mask, i)) continue;
      for (int j = 0; j < n_atoms; ++j) {
        if (in_mask(mask, j) || j == ab || j == ae) continue;
        float dx = u[i][0] - u[j][0], dy = u[i][1] - u[j][1], dz = u[i][2] - u[j][2];
        ++n;
        if (fmaf(dz, dz, fmaf(dy, dy, dx * dx)) < bd2) {
          hit = 1;
          if (early_exit) break;
        }
      }
    }
    bump[p] = (uint8_t)hit;
    pairs[p] = n;
  }
}

/* or_dock_batch plus every restart's final pose in Å: restart_xyz[(atom_off[i] * N + r * A_i + a) * 3 + c] */
int or_dock_batch_poses(int n, const int32_t *atom_off, const float *atom_xyz, const uint8_t *atom_type,
                        const int32_t *frag_off, const int32_t *frag_axis, const uint32_t *frag_mask, const char *ids,
                        const int64_t *id_off, const or_pocket *pocket, const or_config *cfg, int threads,
                        or_result *res, or_restart *rr, uint8_t *tors, float *best_xyz, float *restart_xyz) {
  trig_init();
  or_pk *k = (or_pk *)malloc(sizeof(or_pk));
  if (pk_init(k, pocket)) {
    free(k);
    return -1;
  }
  const int N = cfg->restarts_n;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : 1)
  for (int i = 0; i < n; ++i) {
    or_lig L;
    lig_init(&L, atom_off[i + 1] - atom_off[i], atom_xyz + 3 * (size_t)atom_off[i], atom_type + atom_off[i],
             frag_off[i + 1] - frag_off[i], frag_axis + 2 * (size_t)frag_off[i],
             frag_mask + (size_t)OR_MASK_WORDS * frag_off[i], ids + id_off[i], (size_t)(id_off[i + 1] - id_off[i]));
    dock_ligand_impl(&L, k, cfg, res + i, rr ? rr + (size_t)i * N : NULL, tors ? tors + (size_t)frag_off[i] * N : NULL,
                     best_xyz ? best_xyz + 3 * (size_t)atom_off[i] : NULL, 1,
                     restart_xyz + 3 * (size_t)atom_off[i] * N);
  }
  pk_free(k);
  free(k);
  return 0;
}
