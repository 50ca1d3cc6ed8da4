/*
 * dockscreen.h — C ABI of libdockscreen.so, the B200 (sm_100a) docking hot path.
 *
 * This ABI is the drop-in for the reference package's native slot
 * `dockscreen.kernels._core` (pkg/setup.py:10-18), whose Cython source is absent
 * from the reference (pkg/setup.py:13 names src/dockscreen/kernels/_core.pyx,
 * which does not ship).  By SPEC the slot carries the L2 kernels of Alg. 1
 * that `docking.dock_ligand` and the two
 * engines call.  On B200 the slot is coarser: one call docks
 * a whole packed ligand batch (SPEC.md:277-285 per ligand) with either kernel
 * family of the paper (latency: PAPER.md:287-348, batched: PAPER.md:349-426),
 * and the per-op entry points (ds_op_*) expose the L2 ops themselves.
 *
 * Plain C types only: pointers + sizes, caller-owned host buffers,
 * ctx-owned device memory.  Every function returns DS_OK (0) or a negative
 * DS_ERR_* code; the message of the last failure on the calling thread is
 * available from ds_last_error().  Per-ligand outcomes (NoValidPose,
 * DegenerateAxis: SPEC.md:149, 271, 281) are reported in ds_result.status and
 * never abort a batch.
 *
 * Numeric recipe: DESIGN.md §3 ("pins").  All scores produced here are
 * bit-identical to oracle/ (the CPU restatement) on the same inputs.
 */
#ifndef DOCKSCREEN_H
#define DOCKSCREEN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DS_ABI_VERSION 1

#define DS_MAX_ATOMS 160      /* SPEC.md:44 (largest bucket bound) */
#define DS_MASK_WORDS 5       /* 160 bits of moving mask per fragment           */
#define DS_FRAG_WORDS 8       /* words per packed fragment record (32 B)        */
#define DS_N_TYPES 16         /* element codes 0..15, 0 = hydrogen */
#define DS_MAX_BINS 8
#define DS_MAX_RESTARTS 32
#define DS_TORSION_NONE 255   /* fragment whose angles all bumped (kept as is)  */

/* return codes (SPEC error names in comments) */
enum {
  DS_OK = 0,
  DS_ERR_INVALID_ARG = -1,
  DS_ERR_TOO_MANY_ATOMS = -2,      /* TooManyAtoms */
  DS_ERR_MALFORMED_FRAGMENT = -3,  /* MalformedFragment */
  DS_ERR_INDEX_OUT_OF_RANGE = -4,  /* IndexOutOfRange */
  DS_ERR_DEGENERATE_AXIS = -5,     /* DegenerateAxis */
  DS_ERR_EMPTY_POCKET = -6,        /* EmptyPocket */
  DS_ERR_INFEASIBLE_SHAPE = -7,    /* InfeasibleShape */
  DS_ERR_UNSUPPORTED = -8,
  DS_ERR_CUDA = -9,
  DS_ERR_NO_DEVICE = -10,
  DS_ERR_OOM = -11,
  DS_ERR_PARSE = -12               /* ParseError (malformed .ligq text) */
};

/* per-ligand status in ds_result.status */
enum {
  DS_STATUS_OK = 0,
  DS_STATUS_NO_VALID_POSE = 1,     /* NoValidPose */
  DS_STATUS_DEGENERATE_AXIS = 2,   /* DegenerateAxis      */
  DS_STATUS_NOT_RUN = 3
};

/* kernel families (PAPER.md:287 latency, PAPER.md:349 batched) */
enum { DS_FAMILY_BATCHED = 0, DS_FAMILY_LATENCY = 1 };

typedef struct ds_ctx ds_ctx;
typedef struct ds_pocket ds_pocket;
typedef struct ds_dev_batch ds_dev_batch;

/* Pocket + InteractionTable.  Grid values x-fastest
 * (SPEC.md:472).  Pocket atoms are in Å, same frame as the grid. */
typedef struct ds_pocket_desc {
  float origin[3];
  float spacing;
  int32_t dims[3];
  int32_t n_atoms;
  const int32_t *values;      /* dims[0]*dims[1]*dims[2] */
  const float *atom_xyz;      /* n_atoms*3 */
  const uint8_t *atom_type;   /* n_atoms   */
  const float *table;         /* 16*16, symmetric */
  int32_t n_bins;             /* 1..DS_MAX_BINS */
  const float *bin_ub;        /* ascending upper bounds (Å); last = cutoff */
  const float *bin_mult;
} ds_pocket_desc;

/* DockConfig + the dock seed. */
typedef struct ds_dock_config {
  int32_t restarts_n;          /* N, default 8  */
  int32_t rescore_top_k;       /* K, default 4  */
  int32_t alignment_step_deg;  /* default 12    */
  int32_t torsion_step_deg;    /* default 36    */
  float bump_distance;         /* Å, default 0.8 */
  float similarity_rmsd;       /* Å, default 1.0 */
  float rescore_cutoff;        /* Å, default 8.0 (must equal the last bin_ub) */
  int32_t early_exit;          /* default 1 */
  int64_t seed;                /* dock seed, default 0 */
} ds_dock_config;

/* Packed ligand batch (SoA, CSR over atoms and fragments).
 *  atom_xyzt[4*a+0..2] = centred coordinates d = p - c0 (f32, Å), c0 = f32(f64 mean)
 *  atom_xyzt[4*a+3]    = element code as float (0 = H)
 *  frag_desc[8*f+0..4] = moving-mask bitset over the ligand's atoms
 *  frag_desc[8*f+5]    = axis_begin | axis_end << 8
 *  frag_desc[8*f+6..7] = reserved (0)
 *  id_hash[l]          = FNV-1a-64 of the ligand id bytes (ds_ligand_id_hash)
 *  centroid[3*l]       = c0 (Å) — only used to map output poses back; may be NULL */
typedef struct ds_batch_desc {
  int32_t n_ligands;
  int32_t reserved;
  const int32_t *atom_off;     /* n+1 */
  const float *atom_xyzt;      /* atom_off[n]*4 */
  const int32_t *frag_off;     /* n+1 */
  const uint32_t *frag_desc;   /* frag_off[n]*8 */
  const uint64_t *id_hash;     /* n */
} ds_batch_desc;

/* One result record per ligand (32 B). chem = chem_fx * 2^-24 (DESIGN.md §3 P11). */
typedef struct ds_result {
  int32_t status;
  int32_t geom_score;          /* best pose geometric score */
  int64_t chem_fx;             /* best pose chemical score, fixed point 2^-24 */
  uint8_t best_restart;
  uint8_t best_ax;             /* alignment indices of the best restart (angle = idx*step) */
  uint8_t best_ay;
  uint8_t n_kept;              /* poses kept by select_poses */
  uint32_t poses_scored;
  uint32_t bump_checks;        /* pair evaluations performed (DESIGN.md §3 P14) */
  uint32_t bump_early_exits;
} ds_result;

/* Per (ligand, restart) record, optional. */
typedef struct ds_restart_record {
  int32_t align_score;         /* grid score of the aligned pose */
  int32_t final_geom;          /* grid score after optimize_pose */
  uint8_t ax, ay, valid, kept; /* kept: 1 + keep rank, 0 = not kept */
  int32_t reserved;
} ds_restart_record;

/* Output buffers (caller-owned, host). Everything but `results` may be NULL. */
typedef struct ds_outputs {
  ds_result *results;              /* n */
  float *best_coords;              /* atom_off[n]*3, best pose in Å (pocket frame) */
  uint8_t *best_torsion;           /* frag_off[n], torsion index per fragment of the best pose */
  ds_restart_record *restarts;     /* n*N */
  uint8_t *restart_torsion;        /* frag_off[n]*N, [(frag_off[l]+f)*N + r] */
} ds_outputs;

/* Timing of the last dock call (device-timed with CUDA events on the ctx stream). */
typedef struct ds_stats {
  float total_ms;                  /* first H2D .. last D2H (or kernels only for resident) */
  float align_ms;                  /* alignment kernel(s) */
  float optimize_ms;               /* torsion + select + rescore kernel(s) */
  int32_t launches;                /* kernels launched by the call */
  float select_ms;                 /* batched family: the select + rescore kernel, part of optimize_ms
                                      (0 when the call is chunked and it is not timed separately) */
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  int32_t lat_spread;              /* latency family: CTAs per (ligand, restart) in the optimisation
                                      kernel — 1 = the sequential fragment chain on one SM, n_t = the
                                      cluster-speculative kernel; 0 = batched family */
} ds_stats;

/* ---- library / context -------------------------------------------------- */
int ds_abi_version(void);
const char *ds_last_error(void);
int ds_device_count(int *n);
/* A ctx = one CUDA stream + worst-case workspaces allocated once (PAPER.md:310-313,
 * SPEC.md:394,399).  One ctx per host thread. */
int ds_create(int device, ds_ctx **out);
void ds_destroy(ds_ctx *ctx);
int ds_ctx_alloc_count(const ds_ctx *ctx, int64_t *count);
/* Allocate the worst-case workspace once ("allocate and deallocate that memory
 * only once in the lifetime of the thread"): afterwards ds_dock on batches within these bounds
 * (and the given restarts / alignment step) performs no device or pinned allocation. */
int ds_ctx_reserve(ds_ctx *ctx, int max_ligands, int max_atoms, int max_frags, const ds_dock_config *cfg);
/* Opaque cudaStream_t of the ctx (for external event timing). */
void *ds_ctx_stream(ds_ctx *ctx);
/* Pinned (page-locked) host memory.  Batch arrays and output buffers placed here are
 * DMA'd directly by ds_dock (no staging copy).  NULL on failure. */
void *ds_host_alloc(size_t bytes);
void ds_host_free(void *ptr);
int ds_synchronize(ds_ctx *ctx);

/* ---- pocket ------------------------------------------------------------- */
int ds_pocket_create(ds_ctx *ctx, const ds_pocket_desc *desc, ds_pocket **out);
void ds_pocket_destroy(ds_pocket *pocket);

/* ---- docking (SPEC.md:277 per ligand; engines SPEC.md:391, 401) --------- */
/* Synchronous: H2D of the batch, kernels, D2H of the outputs. */
int ds_dock(ds_ctx *ctx, const ds_pocket *pocket, const ds_batch_desc *batch,
            const ds_dock_config *cfg, int family, const ds_outputs *out, ds_stats *stats);
/* Device-resident variant used for kernel-only timing. */
int ds_batch_upload(ds_ctx *ctx, const ds_batch_desc *batch, ds_dev_batch **out);
int ds_dock_resident(ds_ctx *ctx, const ds_pocket *pocket, ds_dev_batch *batch,
                     const ds_dock_config *cfg, int family, ds_stats *stats);
int ds_batch_download(ds_ctx *ctx, ds_dev_batch *batch, const ds_outputs *out);
void ds_batch_destroy(ds_dev_batch *batch);

/* Engine stream (batched_engine.run; replaces the per-batch ds_dock of the
 * reference's dispatcher): the packed ligand stream of one engine run is kept on the
 * device.  ds_stream_begin sizes it for n_ligands (CSR offsets as in ds_batch_desc, kept by the
 * stream) and zeroes the result records; producers call ds_stream_upload for the ranges [lo, hi)
 * they have packed (base pointers of the WHOLE stream's arrays, ds_pack_ligands layout; pinned
 * memory is DMA'd directly; synchronous, thread-safe for disjoint ranges); a dispatcher docks each
 * batch the bucketizer detaches as a list of stream ligand numbers with ds_stream_dock (its own
 * ctx: stream + scratch; batched family; each ligand at most once per run), and one
 * ds_stream_download returns the records, best poses and best torsion indices of the whole stream
 * (ds_outputs.restarts / restart_torsion must be NULL).  Buffers grow and are kept across runs. */
typedef struct ds_stream ds_stream;
int ds_stream_create(ds_ctx *ctx, ds_stream **out);
void ds_stream_destroy(ds_stream *stream);
int ds_stream_begin(ds_stream *stream, int32_t n_ligands, const int32_t *atom_off, const int32_t *frag_off,
                    int32_t restarts);
int ds_stream_upload(ds_stream *stream, int32_t lo, int32_t hi, const float *atom_xyzt, const uint32_t *frag_desc,
                     const uint64_t *id_hash);
int ds_stream_dock(ds_ctx *ctx, const ds_pocket *pocket, ds_stream *stream, const int32_t *sel, int32_t n_sel,
                   const ds_dock_config *cfg, ds_stats *stats);
int ds_stream_download(ds_ctx *ctx, ds_stream *stream, const ds_outputs *out);

/* Device-side ingest: generate ligands first_index .. first_index +
 * count - 1 of a synthetic dataset (the same ligands as ds_generate_ligands with these shapes,
 * SPEC.md:443 generate_dataset) directly into the ctx's device buffers, packed as ds_pack_ligands
 * would (bit-identical atoms, fragment descriptors and id hashes of "lig_<seed>_<index>"), ready
 * for ds_dock_resident.  Replaces generate + pack + ds_batch_upload (io.generate_batch,
 * native.pack, ResidentBatch in the Python layer).  *device_ms (may be NULL) = the kernel time. */
int ds_generate_resident(ds_ctx *ctx, int64_t seed, int64_t first_index, int32_t count, const int32_t *shapes,
                         ds_dev_batch **out, float *device_ms);
/* Read a resident batch's packed inputs back (any pointer may be NULL): atom_xyzt float[4 * atoms],
 * frag_desc uint32[8 * fragments], id_hash uint64[ligands]. */
int ds_batch_read_inputs(ds_ctx *ctx, const ds_dev_batch *batch, float *atom_xyzt, uint32_t *frag_desc,
                         uint64_t *id_hash);
/* Batch capacity for atom range `range_idx` (0..4) on this device — the B200 analogue of the
 * paper's occupancy-derived batch size (replaces SPEC.md:332 bucket_capacity's
 * fixed A100 numbers): SMs x the smaller resident-warp count of the alignment and torsion kernels
 * (cudaOccupancyMaxActiveBlocksPerMultiprocessor on the kernels themselves; one ligand per warp)
 * x DS_CAPACITY_WAVES (default 2).  The same for every range: the kernels are not
 * range-specialised. */
int ds_query_capacity(ds_ctx *ctx, int range_idx, int *ligands);

/* ---- L2 ops of the native slot, batched on device ------ */
/* grid_score of n_poses poses of n_atoms atoms each, coordinates in Å. */
int ds_op_grid_score(ds_ctx *ctx, const ds_pocket *pocket, const float *coords,
                     int n_atoms, int n_poses, int32_t *out_scores);
/* rescore of n_poses poses; chem in fixed point 2^-24. */
int ds_op_rescore(ds_ctx *ctx, const ds_pocket *pocket, const float *coords,
                  const uint8_t *types, int n_atoms, int n_poses, float cutoff,
                  int64_t *out_chem_fx);

/* apply_rigid of n_poses poses, coordinates in Å: p' = m (p - c) + c with the
 * pinned recipe w = p - c, p'_i = fma(m_i2, w_z, fma(m_i1, w_y, fma(m_i0, w_x, c_i))).  m: 9 floats
 * (row-major) per pose, center: 3 per pose. */
int ds_op_apply_rigid(ds_ctx *ctx, const float *coords, int n_atoms, int n_poses, const float *m,
                      const float *center, float *out);
/* apply_torsion of one fragment (axis atoms, 5-word moving mask) by angle_deg on
 * n_poses poses in Å (DESIGN.md §3 P8, eps = 1e-9 Å); status[p] = 0, or DS_STATUS_DEGENERATE_AXIS
 * with the pose unchanged.  Angle 0 leaves every coordinate bitwise unchanged. */
int ds_op_apply_torsion(ds_ctx *ctx, const float *coords, int n_atoms, int n_poses, int axis_begin,
                        int axis_end, const uint32_t *mask, int angle_deg, float *out, int32_t *status);
/* bump_check of one fragment on n_poses poses in Å (P9, bd2 = f32(bump_distance^2)):
 * bump[p] = 1 iff a moving atom lies closer than bump_distance to a non-moving, non-axis atom;
 * pairs[p] = pair evaluations of the sequential scan (early_exit: up to the first bump). */
int ds_op_bump_check(ds_ctx *ctx, const float *coords, int n_atoms, int n_poses, int axis_begin,
                     int axis_end, const uint32_t *mask, float bump_distance, int early_exit, uint8_t *bump,
                     int64_t *pairs);

/* ---- host-side helpers (input makers and packing; not on the timed path) - */
/* FNV-1a-64 of the id bytes (keys the starting-pose PRNG, DESIGN.md §3 P5). */
uint64_t ds_ligand_id_hash(const char *id, size_t len);
/* Canonical id of generated ligand `index`: "lig_<seed>_<index>"; returns length. */
int ds_generated_id(int64_t seed, int64_t index, char *buf, size_t cap);
/* ids first_index .. first_index + count - 1 of a generated dataset as one blob (no separators)
 * with offsets off[0..count]; buf == NULL fills only off (size query).  Same strings as
 * ds_generated_id. */
int ds_generated_ids(int64_t seed, int64_t first_index, int32_t count, char *buf, int64_t *off);
/* Per-ligand (heavy, frags) shapes of the mixed datasets (BASELINE configs 3, 5):
 * heavy ~ U{heavy_min..heavy_max}, frags ~ U{0..min(frag_max, heavy-2)}. */
int ds_mixed_shapes(int64_t seed, int64_t first_index, int32_t count, int32_t heavy_min,
                    int32_t heavy_max, int32_t frag_max, int32_t *shapes /* 2*count */);
/* SPEC.md:443 generate_dataset for ligands first_index .. first_index+count-1.
 * shapes[2i], shapes[2i+1] = (heavy atoms, fragments).  Pass 1 (atom_xyz == NULL)
 * fills the three CSR offset arrays (count+1 each); pass 2 fills the payload.
 * Coordinates are absolute (Å).  Bonds/axes are ligand-local atom indices. */
int ds_generate_ligands(int64_t seed, int64_t first_index, int32_t count, const int32_t *shapes,
                        int32_t *atom_off, int32_t *bond_off, int32_t *frag_off,
                        float *atom_xyz, uint8_t *atom_type, int32_t *bonds,
                        int32_t *frag_axis, uint32_t *frag_mask /* 5 words per fragment */);
/* Pack ligands into the ds_batch_desc layout (validating SPEC.md:81-89 except the
 * bond-cut rule, which needs bonds).  id_hash is an input when ids == NULL. On an
 * invalid ligand returns its DS_ERR_* code and sets *bad_index. */
int ds_pack_ligands(int32_t count, const int32_t *atom_off, const float *atom_xyz,
                    const uint8_t *atom_type, const int32_t *frag_off, const int32_t *frag_axis,
                    const uint32_t *frag_mask, const char *ids, const int64_t *id_off,
                    float *atom_xyzt, uint32_t *frag_desc, uint64_t *id_hash, float *centroid,
                    int32_t *bad_index);
/* Synthetic pocket atoms: uniform in the shell rmin <= r <= rmax, types 1..15. */
int ds_generate_pocket_atoms(int64_t seed, int32_t n, float rmin, float rmax,
                             float *atom_xyz, uint8_t *atom_type);
/* SPEC.md:453 build_pocket grid (x-fastest).  values == NULL: size query. */
int ds_build_pocket_grid(const float *atom_xyz, int32_t n_atoms, float spacing, float padding,
                         float origin[3], int32_t dims[3], int32_t *values);
/* The same grid built on the ctx's device (thread per node; bit-identical to ds_build_pocket_grid,
 * DESIGN.md §3 P18).  values: host buffer of dims[0]*dims[1]*dims[2] int32 (query the size with
 * ds_build_pocket_grid(..., NULL) first); device_ms (optional): kernel time.  SURVEY §8(f) rank 2. */
int ds_build_pocket_grid_device(ds_ctx *ctx, const float *atom_xyz, int32_t n_atoms, float spacing,
                                float padding, float origin[3], int32_t dims[3], int32_t *values,
                                float *device_ms);
/* Native .ligq parser (io.parse_ligand_file): molecules parsed and validated
 * (validate_ligand) in parallel, kept in file order.  ds_ligq_parse returns counts
 * {ligands, atoms, bonds, fragments, id bytes, skipped invalid} and a handle; ds_ligq_fill copies
 * the CSR batch into caller arrays (offset arrays have ligands + 1 entries); ds_ligq_free.  Errors:
 * DS_ERR_PARSE (message in err) or the validation code of the first invalid molecule unless
 * skip_invalid. */
typedef struct ds_ligq ds_ligq;
int ds_ligq_parse(const char *text, int64_t len, int32_t skip_invalid, ds_ligq **out, int64_t counts[6],
                  char *err, int32_t err_len);
int ds_ligq_fill(const ds_ligq *h, int32_t *atom_off, float *atom_xyz, uint8_t *atom_type, int32_t *bond_off,
                 int32_t *bonds, int32_t *frag_off, int32_t *frag_axis, uint32_t *frag_mask, char *ids,
                 int64_t *id_off);
void ds_ligq_free(ds_ligq *h);
/* validate_ligand over a CSR batch of the reference's objects: element types as
 * int64 (any value), is_heavy flags, bonds, fragment axes and the moving atoms as a CSR list
 * (mv_off has fragments + 1 entries, absolute into mv).  codes[i] = 0 or the DS_ERR_* of ligand i. */
int ds_validate_ligands(int32_t n, const int32_t *atom_off, const int64_t *atom_type, const uint8_t *is_heavy,
                        const int32_t *bond_off, const int32_t *bonds, const int32_t *frag_off,
                        const int32_t *frag_axis, const int64_t *mv_off, const int64_t *mv, int32_t *codes);
/* Rows sel[0..n_sel) of a CSR array (src_off: rows + 1 offsets, elem_bytes per element) gathered
 * into dst in selection order: pass 1 (dst == NULL) fills dst_off[n_sel + 1].  Used by the batched
 * engine to cut a bucket's batch out of the packed stream (bucketizer.push). */
int ds_csr_gather(int32_t n_sel, const int32_t *sel, const int32_t *src_off, const void *src, int32_t elem_bytes,
                  int32_t *dst_off, void *dst);
/* Inverse: row k of src goes to row sel[k] of dst (offsets dst_off) — per-ligand outputs of a
 * batch back into stream order (EngineReport). */
int ds_csr_scatter(int32_t n_sel, const int32_t *sel, const int32_t *src_off, const void *src, int32_t elem_bytes,
                   const int32_t *dst_off, void *dst);
/* Seeded symmetric 16x16 interaction table in [-1, 1]. */
/* Threads of the host-side parallel loops (packing, validation, generation) run by the CALLING
 * thread from now on; concurrent producer threads split the host cores instead of each spawning a
 * team of all of them. */
int ds_set_host_threads(int32_t n);
int ds_default_table(int64_t seed, float *table /* 256 */);

#ifdef __cplusplus
}
#endif
#endif /* DOCKSCREEN_H */
