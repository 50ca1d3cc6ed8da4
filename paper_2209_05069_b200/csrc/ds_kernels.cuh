// Kernel parameter blocks shared by ds_kernels.cu and ds_api.cu.
#pragma once
#include "ds_device.cuh"

namespace ds {

struct PocketView {
  const uint8_t *grid;       // (nx+2)(ny+2)(nz+2) values + 128 (uint8), x-fastest, halo = kOutside
  GridGeom g;
  int grid_bytes;            // rounded up to 16 B
  float inv_s, spacing;
  float ox, oy, oz;
  int n_atoms;
  const float4 *patoms;      // pocket atoms in the grid frame, .w = element code
  const int32_t *wfx;        // [16][16][nb+1] fixed-point table*mult (2^-24); entry nb = 0
  int part_terms;            // weight terms an int32 partial sum can hold without overflow:
                             // floor((2^31 - 1) / max |W|) (2^7 for the default table)
  int nb;
  float ub2[DS_MAX_BINS];    // squared bin upper bounds, grid frame
  // bin look-up table, exact when every ub2 has its low lut_shift bits zero (the defaults do):
  // bin = bin_lut[min(bits(d2) >> lut_shift, lut_cap)]; lut_cap < 0: no table (compare path)
  const uint8_t *bin_lut;
  int lut_shift, lut_cap;
  int lut_full;              // the table covers every non-negative float (lut_cap = 0x7FFFFFFF >> shift)
  const float2 *trig;        // (cos, sin) of integer degrees 0..359 (f32 of f64)
};

struct BatchView {
  int L;
  const int *atom_off;       // L+1
  const float4 *atoms;       // centred coords + type
  const int *frag_off;       // L+1
  const uint4 *frags;        // 2 uint4 per fragment (mask words 0..4, axis word 5)
  const uint64_t *idh;
};

struct DockParams {
  int N, K;
  int n_a, step_a, n_rot;
  int n_t, step_t;
  int64_t seed;
  int early_exit;
  float bd2;                 // squared bump distance, grid frame
  float eps_axis;            // DegenerateAxis threshold, grid frame
  double thr2;               // squared similarity RMSD, grid frame
  float cull2;               // squared bump-candidate bound (bump distance + 0.02 nodes), grid frame
  float cull_r;              // the bound itself (rounded up), for the per-fragment (h, r) box
  int slot_atoms;            // batched select: pose-slot stride (the launch's largest ligand)
  unsigned opaque0;          // always 0: XORed into loop-invariant index terms so ptxas keeps them as
                             // ALU adds instead of re-deriving them with FMA-pipe IMADs
  // torsion sweep lane layout of the first angle block (angles 0 .. min(32, n_t) - 1): lane ->
  // a | gi << 8 | (gi < G) << 16, and the mask of the lanes sharing its angle (no divisions on device)
  unsigned sweep_lane[32];
  unsigned sweep_same[32];
};

struct AlignOut {
  uint32_t *keys;            // L*N packed (score+32768)<<16 | (65535-rot)
};

struct OptOut {
  ds_result *res;            // L
  ds_restart_record *rrec;   // L*N (may be null)
  uint8_t *rtors;            // frag_total*N (always)
  float4 *final_u;           // final poses. latency: (lig*N + r)*DS_MAX_ATOMS; batched: per ligand,
                             // ((atom_off - atom_base)*N + r*A)
  int *rgv;                  // batched: L*N (final geom << 1) | valid
  long long atom_base;       // batched: first atom of the launch range
  float *best_coords;        // atom_total*3 (may be null)
  uint8_t *best_tors;        // frag_total (may be null)
  uint8_t *rtors_host;       // latency, zero-copy outputs: the last CTA copies its ligand's rtors here
  const int *sel_order;      // batched select: queue item -> ligand (an engine stream's batch), null = identity
};

}  // namespace ds
