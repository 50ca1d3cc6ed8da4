// C ABI of libdockscreen (include/dockscreen.h): contexts, pocket upload, batch docking.
//
// The context is the paper's latency-implementation unit: one host thread,
// one CUDA stream, worst-case device workspace allocated once and reused.  Batched docking
// reuses the same context; its buffers grow geometrically with the batch.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "ds_kernels.cuh"

namespace ds {
int align_warp_smem_bytes_host(int N);
void launch_align_batched(const PocketView &pk, const BatchView &bt, const DockParams &dp, const int *order,
                          AlignOut out, int *queue, int grid_in_smem, int blocks, int warps, size_t smem,
                          cudaStream_t st);
void launch_torsion_batched(const PocketView &pk, const BatchView &bt, const DockParams &dp, const int *order,
                            const uint32_t *keys, OptOut out, int *queue, int blocks, cudaStream_t st);
void launch_select_batched(const PocketView &pk, const BatchView &bt, const DockParams &dp, const uint32_t *keys,
                           OptOut out, int *queue, int sm_count, size_t smem_optin, cudaStream_t st);
size_t select_cta_smem_bytes(int n_patoms, int nb, int lut_cap, int K, int slot_atoms);
int torsion_blocks_per_sm();
int select_blocks_per_sm(size_t smem);
int align_blocks_per_sm(int warps, size_t smem);
bool launch_align_latency(const PocketView &pk, const BatchView &bt, const DockParams &dp, int max_atoms, int *scores,
                          unsigned *keys, cudaStream_t st);
size_t latency_rec_bytes();
void launch_generate_ligands(long long seed, long long first_index, int count, const int *shapes, const int *atom_off,
                             const int *frag_off, float4 *atoms, uint32_t *frag_desc, uint64_t *id_hash, int sm_count,
                             cudaStream_t st);
void launch_build_pocket(const float *atom_xyz, int P, const double *origin, double s, const int *dims,
                         int32_t *values, int sm_count, cudaStream_t st);
void launch_optimize_latency(const PocketView &pk, const BatchView &bt, const DockParams &dp, int *scores,
                             const unsigned *keys, OptOut out, void *recs, int *done, bool pdl, cudaStream_t st);
bool launch_spread_latency(const PocketView &pk, const BatchView &bt, const DockParams &dp, OptOut out, void *recs,
                           int *done, cudaStream_t st);
void launch_grid_score(const PocketView &pk, const float *coords, int n_atoms, int n_poses, int32_t *out,
                       cudaStream_t st);
void launch_rescore(const PocketView &pk, const float *coords, const uint8_t *types, int n_atoms, int n_poses,
                    float cutoff2, int64_t *out, cudaStream_t st);
void launch_apply_rigid(const float *coords, int n_atoms, int n_poses, const float *m, const float *center, float *out,
                        cudaStream_t st);
void launch_apply_torsion(const float *coords, int n_atoms, int n_poses, int ab, int ae, const uint32_t *mask,
                          float2 cs, int identity, float *out, int32_t *status, cudaStream_t st);
void launch_bump_check(const float *coords, int n_atoms, int n_poses, int ab, int ae, const uint32_t *mask, float bd2,
                       int early_exit, uint8_t *bump, long long *pairs, cudaStream_t st);
}  // namespace ds

using namespace ds;

namespace {
thread_local char g_err[512];

int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

#define DS_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) return fail(DS_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

// API entry: make the context's device current and drop any non-sticky error left in this thread
// by an earlier, unrelated runtime call, so the launch checks below report only this call's errors
cudaError_t enter_device(int device) {
  cudaGetLastError();
  const cudaError_t e = cudaSetDevice(device);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// device buffer that grows geometrically; counts cudaMalloc calls
struct DevBuf {
  void *p = nullptr;
  size_t cap = 0;
};
}  // namespace

struct ds_ctx {
  int device = 0;
  int sm_count = 0;
  size_t smem_optin = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy = nullptr;      // H2D/D2H of the chunked ds_dock pipeline
  std::vector<cudaEvent_t> pev;     // pipeline events (4 per chunk)
  cudaEvent_t ev[6] = {};
  int64_t allocs = 0;
  // generation of the per-array batch buffers: bumped by every call that may overwrite or
  // reallocate them; a resident batch handle is valid only while its stamp is current
  uint64_t gen = 1;
  float2 *trig = nullptr;       // 360 (cos, sin)
  // batch-sized device buffers
  DevBuf b_atom_off, b_atoms, b_frag_off, b_frags, b_idh, b_order_a, b_order_o, b_keys, b_res, b_rrec, b_rtors,
      b_coords, b_btors, b_queue, b_scratch, b_rgv, b_lat_scores, b_lat_recs, b_lat_done;
  // device pointers of the batch being docked: the per-array buffers above, or for small calls
  // (ds_dock "express" path) two arenas moved with one H2D and one D2H each
  struct IoView {
    int *atom_off;
    float4 *atoms;
    int *frag_off;
    uint4 *frags;
    uint64_t *idh;
    int *order_a, *order_o;
    ds_result *res;
    ds_restart_record *rrec;
    uint8_t *rtors;
    float *coords;
    uint8_t *btors;
  } io{};
  DevBuf x_in, x_out;
  DevBuf op_in, op_aux, op_out;   // the ds_op_* entry points (never touch a resident batch)
  // latency-family scratch (alignment scores, per-ligand done counters) is left zeroed by the
  // kernels; cleared here only after a (re)allocation or a failed call
  bool lat_pdl = false;
  bool lat_dirty = true;
  void *lat_scores_seen = nullptr, *lat_done_seen = nullptr;
  size_t x_in_bytes = 0, x_out_bytes = 0, x_out_off[5] = {};
  // express latency calls write their outputs straight into the pinned staging buffer (zero-copy,
  // no D2H); x_rtors_host is where the last CTA copies the per-restart torsion indices
  bool x_zero_copy = false;
  uint8_t *x_rtors_host = nullptr;
  // during ds_stream_dock only: the engine stream's per-(ligand, restart) keys and (geom, valid)
  // words (indexed by the stream's ligand numbers) and the batch's select order; null otherwise
  uint32_t *sv_keys = nullptr;
  int *sv_rgv = nullptr;
  const int *sv_sel = nullptr;
  // pinned host staging
  void *h_stage = nullptr;
  size_t h_cap = 0;
  int ensure(DevBuf &b, size_t bytes) {
    if (bytes <= b.cap) return DS_OK;
    size_t nc = std::max(bytes, b.cap * 3 / 2);
    nc = (nc + 255) & ~(size_t)255;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
    cudaError_t e = cudaMalloc(&b.p, nc);
    if (e != cudaSuccess) return fail(DS_ERR_OOM, "cudaMalloc(%zu): %s", nc, cudaGetErrorString(e));
    b.cap = nc;
    ++allocs;
    return DS_OK;
  }
  int ensure_host(size_t bytes) {
    if (bytes <= h_cap) return DS_OK;
    size_t nc = std::max(bytes, h_cap * 3 / 2);
    if (h_stage) cudaFreeHost(h_stage);
    h_stage = nullptr;
    h_cap = 0;
    cudaError_t e = cudaMallocHost(&h_stage, nc);
    if (e != cudaSuccess) return fail(DS_ERR_OOM, "cudaMallocHost(%zu): %s", nc, cudaGetErrorString(e));
    h_cap = nc;
    ++allocs;
    return DS_OK;
  }
};

struct ds_pocket {
  ds_ctx *ctx = nullptr;        // creating context (not dereferenced after creation)
  int device = 0;               // its device: the pocket may outlive the context
  PocketView view{};
  uint8_t *d_grid = nullptr;
  uint8_t *d_lut = nullptr;
  float4 *d_patoms = nullptr;
  int32_t *d_wfx = nullptr;
  float cutoff = 0.f;
};

struct ds_dev_batch {
  ds_ctx *ctx = nullptr;
  uint64_t gen = 0;             // ds_ctx::gen when the batch was placed in the ctx's buffers
  int L = 0, n_atoms = 0, n_frags = 0;
  int N = 0;
  std::vector<int> atom_off, frag_off;  // host copies for downloads
  bool docked = false;
};

extern "C" {

int ds_abi_version(void) { return DS_ABI_VERSION; }
const char *ds_last_error(void) { return g_err; }

int ds_device_count(int *n) {
  if (!n) return fail(DS_ERR_INVALID_ARG, "n is NULL");
  cudaError_t e = cudaGetDeviceCount(n);
  if (e != cudaSuccess) {
    *n = 0;
    return fail(DS_ERR_NO_DEVICE, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  return DS_OK;
}

int ds_create(int device, ds_ctx **out) {
  if (!out) return fail(DS_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return fail(DS_ERR_NO_DEVICE, "no CUDA device visible");
  if (device < 0 || device >= n) return fail(DS_ERR_INVALID_ARG, "device %d out of range (%d devices)", device, n);
  DS_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  DS_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(DS_ERR_UNSUPPORTED, "libdockscreen is built for sm_100a; device is sm_%d%d", prop.major, prop.minor);
  ds_ctx *c = new ds_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  c->smem_optin = prop.sharedMemPerBlockOptin;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return fail(DS_ERR_CUDA, "cudaStreamCreate failed");
  }
  for (auto &e : c->ev) cudaEventCreate(&e);
  // P0: trig table of integer degrees, f32 of f64 (shared by every kernel)
  float2 h[360];
  for (int d = 0; d < 360; ++d) {
    const double rad = (double)d * 0.017453292519943295;  // pi/180
    h[d] = make_float2((float)cos(rad), (float)sin(rad));
  }
  if (cudaMalloc(&c->trig, sizeof h) != cudaSuccess) {
    ds_destroy(c);
    return fail(DS_ERR_OOM, "cudaMalloc(trig) failed");
  }
  ++c->allocs;
  cudaMemcpy(c->trig, h, sizeof h, cudaMemcpyHostToDevice);
  *out = c;
  return DS_OK;
}

void ds_destroy(ds_ctx *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  DevBuf *bufs[] = {&c->b_atom_off, &c->b_atoms, &c->b_frag_off, &c->b_frags, &c->b_idh, &c->b_order_a,
                    &c->b_order_o, &c->b_keys, &c->b_res, &c->b_rrec, &c->b_rtors, &c->b_coords, &c->b_btors,
                    &c->b_queue, &c->b_scratch, &c->b_rgv, &c->b_lat_scores, &c->b_lat_recs, &c->b_lat_done,
                    &c->x_in, &c->x_out, &c->op_in, &c->op_aux, &c->op_out};
  for (DevBuf *b : bufs)
    if (b->p) cudaFree(b->p);
  if (c->trig) cudaFree(c->trig);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  for (auto &e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto &e : c->pev)
    if (e) cudaEventDestroy(e);
  if (c->copy) cudaStreamDestroy(c->copy);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int ds_ctx_alloc_count(const ds_ctx *c, int64_t *count) {
  if (!c || !count) return fail(DS_ERR_INVALID_ARG, "NULL argument");
  *count = c->allocs;
  return DS_OK;
}

void *ds_ctx_stream(ds_ctx *c) { return c ? (void *)c->stream : nullptr; }

void *ds_host_alloc(size_t bytes) {
  void *p = nullptr;
  if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    fail(DS_ERR_OOM, "cudaHostAlloc(%zu) failed", bytes);
    return nullptr;
  }
  return p;
}

void ds_host_free(void *p) {
  if (p) cudaFreeHost(p);
}

int ds_synchronize(ds_ctx *c) {
  if (!c) return fail(DS_ERR_INVALID_ARG, "NULL ctx");
  DS_CUDA(cudaStreamSynchronize(c->stream));
  return DS_OK;
}

int ds_pocket_create(ds_ctx *c, const ds_pocket_desc *d, ds_pocket **out) {
  if (!c || !d || !out) return fail(DS_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  if (!(d->spacing > 0.f)) return fail(DS_ERR_INVALID_ARG, "grid spacing must be > 0");
  for (int k = 0; k < 3; ++k)
    if (d->dims[k] < 1 || d->dims[k] >= (1 << 21)) return fail(DS_ERR_INVALID_ARG, "bad grid dims");
  const int64_t G = (int64_t)d->dims[0] * d->dims[1] * d->dims[2];
  if (G >= (1ll << 30)) return fail(DS_ERR_UNSUPPORTED, "grid too large");
  if (!d->values) return fail(DS_ERR_INVALID_ARG, "grid values NULL");
  if (d->n_atoms < 0 || (d->n_atoms > 0 && (!d->atom_xyz || !d->atom_type)))
    return fail(DS_ERR_INVALID_ARG, "bad pocket atoms");
  if (d->n_atoms > 4096) return fail(DS_ERR_UNSUPPORTED, "at most 4096 pocket atoms (staged in shared memory)");
  if (!d->table || d->n_bins < 1 || d->n_bins > DS_MAX_BINS || !d->bin_ub || !d->bin_mult)
    return fail(DS_ERR_INVALID_ARG, "bad interaction table");
  for (int b = 1; b < d->n_bins; ++b)
    if (!(d->bin_ub[b] > d->bin_ub[b - 1])) return fail(DS_ERR_INVALID_ARG, "bins must be ascending");
  // int8 device grid with a one-node halo of kOutside: every value must fit
  const int64_t NX = d->dims[0] + 2, NY = d->dims[1] + 2, NZ = d->dims[2] + 2;
  const int gbytes = (int)((NX * NY * NZ + 15) & ~15ll);
  std::vector<uint8_t> g8(gbytes, (uint8_t)(kOutside + 128));  // stored biased by +128
  for (int64_t z = 0; z < d->dims[2]; ++z)
    for (int64_t y = 0; y < d->dims[1]; ++y)
      for (int64_t x = 0; x < d->dims[0]; ++x) {
        const int32_t val = d->values[x + d->dims[0] * (y + d->dims[1] * z)];
        if (val < -128 || val > 127)
          return fail(DS_ERR_UNSUPPORTED, "grid value %d does not fit int8", val);
        g8[(x + 1) + NX * ((y + 1) + NY * (z + 1))] = (uint8_t)(val + 128);
      }
  for (int t = 0; t < DS_N_TYPES * DS_N_TYPES; ++t)
    if (d->table[t] != d->table[(t % DS_N_TYPES) * DS_N_TYPES + t / DS_N_TYPES])
      return fail(DS_ERR_INVALID_ARG, "interaction table must be symmetric");
  DS_CUDA(enter_device(c->device));
  ds_pocket *p = new ds_pocket();
  p->ctx = c;
  p->device = c->device;
  PocketView &v = p->view;
  v.g.nx = d->dims[0];
  v.g.ny = d->dims[1];
  v.g.nz = d->dims[2];
  v.g.bx = (unsigned)(NX - 1);
  v.g.by = (unsigned)(NY - 1);
  v.g.bz = (unsigned)(NZ - 1);
  v.g.NX = (unsigned)NX;
  v.g.NXY = (unsigned)(NX * NY);
  v.grid_bytes = gbytes;
  v.spacing = d->spacing;
  v.inv_s = (float)(1.0 / (double)d->spacing);  // P2
  v.ox = d->origin[0];
  v.oy = d->origin[1];
  v.oz = d->origin[2];
  v.n_atoms = d->n_atoms;
  v.nb = d->n_bins;
  for (int b = 0; b < DS_MAX_BINS; ++b) {
    const double ub = b < d->n_bins ? (double)d->bin_ub[b] / (double)d->spacing : 0.0;
    v.ub2[b] = (float)(ub * ub);  // P11
  }
  p->cutoff = d->bin_ub[d->n_bins - 1];
  // exact bin LUT (P11): with S = the common count of trailing zero bits of the squared bounds,
  // d2 >= ub2_b  <=>  bits(d2) >> S >= bits(ub2_b) >> S  for every d2 >= +0 (and NaN -> beyond)
  std::vector<uint8_t> lut;
  {
    int S = 23;
    for (int b = 0; b < d->n_bins; ++b) {
      uint32_t u;
      memcpy(&u, &v.ub2[b], 4);
      if (u) S = std::min(S, __builtin_ctz(u));
    }
    uint32_t ul;
    memcpy(&ul, &v.ub2[d->n_bins - 1], 4);
    // full range when it is small: every non-negative float's bits >> S index the table directly
    // (no clamp in the kernels); else entries up to the last bound and a clamp
    const uint32_t full = 0x7FFFFFFFu >> S;
    v.lut_full = full < 4096;
    const uint32_t cap = v.lut_full ? full : ul >> S;
    v.lut_shift = S;
    v.lut_cap = -1;
    if (cap < 4096) {
      lut.resize(cap + 1);
      for (uint32_t k = 0; k <= cap; ++k) {
        int n = 0;
        for (int b = 0; b < d->n_bins; ++b) {
          uint32_t u;
          memcpy(&u, &v.ub2[b], 4);
          n += (u >> S) <= k;
        }
        lut[k] = (uint8_t)n;
      }
      v.lut_cap = (int)cap;
    }
  }
  // pocket atoms in the grid frame: f32((p - o) / s) evaluated in f64 (P11)
  std::vector<float4> pa(std::max(d->n_atoms, 1));
  for (int j = 0; j < d->n_atoms; ++j) {
    float q[3];
    for (int k = 0; k < 3; ++k)
      q[k] = (float)(((double)d->atom_xyz[3 * j + k] - (double)d->origin[k]) / (double)d->spacing);
    if (d->atom_type[j] >= DS_N_TYPES) {
      delete p;
      return fail(DS_ERR_INDEX_OUT_OF_RANGE, "pocket atom %d type %d", j, d->atom_type[j]);
    }
    pa[j] = make_float4(q[0], q[1], q[2], (float)d->atom_type[j]);
  }
  // fixed-point table x multiplier: W = llrint(f32(table*mult) * 2^24), bin nb -> 0 (P11)
  const int nb1 = d->n_bins + 1;
  std::vector<int32_t> w((size_t)DS_N_TYPES * DS_N_TYPES * nb1, 0);
  for (int t = 0; t < DS_N_TYPES * DS_N_TYPES; ++t)
    for (int b = 0; b < d->n_bins; ++b) {
      const float prod = d->table[t] * d->bin_mult[b];
      const double s = (double)prod * 16777216.0;
      if (!(fabs(s) < 2147483647.0)) {
        delete p;
        return fail(DS_ERR_UNSUPPORTED, "table*multiplier %g out of fixed-point range", (double)prod);
      }
      w[(size_t)t * nb1 + b] = (int32_t)llrint(s);
    }
  {
    int64_t wmax = 1;
    for (int32_t x : w) wmax = std::max<int64_t>(wmax, x < 0 ? -(int64_t)x : (int64_t)x);
    v.part_terms = (int)std::min<int64_t>((int64_t)INT32_MAX / wmax, 1 << 30);
  }
  v.trig = c->trig;
  if (cudaMalloc(&p->d_grid, gbytes) != cudaSuccess || cudaMalloc(&p->d_patoms, pa.size() * sizeof(float4)) != cudaSuccess ||
      cudaMalloc(&p->d_wfx, w.size() * 4) != cudaSuccess) {
    ds_pocket_destroy(p);
    return fail(DS_ERR_OOM, "pocket allocation failed");
  }
  c->allocs += 3;
  if (!lut.empty()) {
    if (cudaMalloc(&p->d_lut, lut.size()) != cudaSuccess) {
      ds_pocket_destroy(p);
      return fail(DS_ERR_OOM, "pocket allocation failed");
    }
    c->allocs += 1;
    cudaMemcpy(p->d_lut, lut.data(), lut.size(), cudaMemcpyHostToDevice);
  }
  v.bin_lut = p->d_lut;
  cudaMemcpy(p->d_grid, g8.data(), gbytes, cudaMemcpyHostToDevice);
  cudaMemcpy(p->d_patoms, pa.data(), pa.size() * sizeof(float4), cudaMemcpyHostToDevice);
  cudaMemcpy(p->d_wfx, w.data(), w.size() * 4, cudaMemcpyHostToDevice);
  v.grid = p->d_grid;
  v.patoms = p->d_patoms;
  v.wfx = p->d_wfx;
  // keep the grid L2-resident for the LDG paths (access-policy window, north star)
  cudaStreamAttrValue attr = {};
  size_t maxwin = 0;
  int l2max = 0;
  cudaDeviceGetAttribute(&l2max, cudaDevAttrMaxAccessPolicyWindowSize, c->device);
  maxwin = (size_t)l2max;
  if (maxwin > 0) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min((size_t)gbytes, (size_t)64 << 20));
    attr.accessPolicyWindow.base_ptr = p->d_grid;
    attr.accessPolicyWindow.num_bytes = std::min((size_t)gbytes, maxwin);
    attr.accessPolicyWindow.hitRatio = 1.0f;
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    ds_pocket_destroy(p);
    return fail(DS_ERR_CUDA, "pocket upload: %s", cudaGetErrorString(e));
  }
  *out = p;
  return DS_OK;
}

void ds_pocket_destroy(ds_pocket *p) {
  if (!p) return;
  cudaSetDevice(p->device);
  if (p->d_grid) cudaFree(p->d_grid);
  if (p->d_patoms) cudaFree(p->d_patoms);
  if (p->d_wfx) cudaFree(p->d_wfx);
  if (p->d_lut) cudaFree(p->d_lut);
  delete p;
}

}  // extern "C"

namespace {

int check_config(const ds_dock_config *cfg, const ds_pocket *pk, DockParams *dp) {
  if (!cfg) return fail(DS_ERR_INVALID_ARG, "cfg is NULL");
  if (cfg->restarts_n < 1 || cfg->restarts_n > DS_MAX_RESTARTS)
    return fail(DS_ERR_INVALID_ARG, "restarts_n must be in 1..%d", DS_MAX_RESTARTS);
  if (cfg->rescore_top_k < 1 || cfg->rescore_top_k > cfg->restarts_n)
    return fail(DS_ERR_INVALID_ARG, "rescore_top_k must be in 1..restarts_n");
  if (cfg->alignment_step_deg < 1 || 360 % cfg->alignment_step_deg)
    return fail(DS_ERR_INVALID_ARG, "360 must be divisible by alignment_step_deg");
  if (cfg->torsion_step_deg < 1 || 360 % cfg->torsion_step_deg)
    return fail(DS_ERR_INVALID_ARG, "360 must be divisible by torsion_step_deg");
  if (!(cfg->bump_distance > 0.f) || !(cfg->similarity_rmsd > 0.f) || !(cfg->rescore_cutoff > 0.f))
    return fail(DS_ERR_INVALID_ARG, "distances must be positive");
  if (cfg->rescore_cutoff != pk->cutoff)
    return fail(DS_ERR_INVALID_ARG, "rescore_cutoff %g must equal the last bin bound %g (SPEC.md:179)",
                (double)cfg->rescore_cutoff, (double)pk->cutoff);
  dp->N = cfg->restarts_n;
  dp->K = cfg->rescore_top_k;
  dp->step_a = cfg->alignment_step_deg;
  dp->n_a = 360 / cfg->alignment_step_deg;
  dp->n_rot = dp->n_a * dp->n_a;
  if (dp->n_rot > 65536) return fail(DS_ERR_UNSUPPORTED, "alignment_step_deg >= 2 required on device (32-bit argmax keys)");
  dp->step_t = cfg->torsion_step_deg;
  dp->n_t = 360 / cfg->torsion_step_deg;
  dp->seed = cfg->seed;
  dp->early_exit = cfg->early_exit ? 1 : 0;
  const double s = (double)pk->view.spacing;
  const double bd = (double)cfg->bump_distance / s;
  dp->bd2 = (float)(bd * bd);                              // P9
  dp->eps_axis = (float)(1e-9 / s);                        // P8
  const double th = (double)cfg->similarity_rmsd / s;
  dp->thr2 = th * th;                                      // P12
  dp->cull2 = (float)((bd + 0.02) * (bd + 0.02));          // conservative bump-candidate bound
  dp->cull_r = (float)((bd + 0.02) * (1.0 + 1e-6));
  dp->opaque0 = 0u;
  {
    const int nA = std::min(32, dp->n_t), G = 32 / nA;
    for (int l = 0; l < 32; ++l) {
      const int a = l % nA, gi = l / nA;
      unsigned same = 0;
      for (int t = 0; t < G; ++t) same |= 1u << (a + t * nA);
      dp->sweep_lane[l] = (unsigned)a | ((unsigned)gi << 8) | ((unsigned)(gi < G) << 16);
      dp->sweep_same[l] = same;
    }
  }
  return DS_OK;
}

int check_batch(const ds_batch_desc *b) {
  if (!b) return fail(DS_ERR_INVALID_ARG, "batch is NULL");
  if (b->n_ligands < 0) return fail(DS_ERR_INVALID_ARG, "n_ligands < 0");
  if (b->n_ligands == 0) return DS_OK;
  if (!b->atom_off || !b->atom_xyzt || !b->frag_off || !b->id_hash)
    return fail(DS_ERR_INVALID_ARG, "batch arrays NULL");
  if (b->frag_off[b->n_ligands] > 0 && !b->frag_desc) return fail(DS_ERR_INVALID_ARG, "frag_desc NULL");
  // the scan is O(atoms + fragments) over host memory (tens of MB for a 200k-ligand batch): run it
  // on all host threads, then report the lowest failing ligand exactly as the serial scan would
  auto bad = [b](int i) {
    const int A = b->atom_off[i + 1] - b->atom_off[i];
    if (A < 1 || A > DS_MAX_ATOMS || b->frag_off[i + 1] < b->frag_off[i]) return true;
    for (int f = b->frag_off[i]; f < b->frag_off[i + 1]; ++f) {
      const uint32_t ax = b->frag_desc[(size_t)DS_FRAG_WORDS * f + 5];
      if ((int)(ax & 0xFF) >= A || (int)((ax >> 8) & 0xFF) >= A) return true;
    }
    return false;
  };
  int first = b->n_ligands;
#pragma omp parallel for schedule(static) reduction(min : first) if (b->n_ligands >= 4096)
  for (int i = 0; i < b->n_ligands; ++i)
    if (i < first && bad(i)) first = i;
  if (first < b->n_ligands) {
    const int i = first;
    const int A = b->atom_off[i + 1] - b->atom_off[i];
    if (A < 1) return fail(DS_ERR_INVALID_ARG, "ligand %d has no atoms", i);
    if (A > DS_MAX_ATOMS) return fail(DS_ERR_TOO_MANY_ATOMS, "ligand %d has %d atoms (> %d)", i, A, DS_MAX_ATOMS);
    if (b->frag_off[i + 1] < b->frag_off[i]) return fail(DS_ERR_INVALID_ARG, "frag_off not monotone");
    return fail(DS_ERR_INDEX_OUT_OF_RANGE, "ligand %d fragment axis out of range", i);
  }
  return DS_OK;
}

// LPT orders: alignment work ~ A (counting sort, descending); optimisation work ~ F*(A^2)/4 + A
// LPT orders of ligands [L0, L1) as indices relative to L0, written to oa/oo (L1-L0 entries each)
void lpt_orders_range(const ds_batch_desc *b, int L0, int L1, int *oa, int *oo) {
  const int L = L1 - L0;
  // counting sorts, descending cost: alignment ~ A, optimisation ~ (F + 2) * A (torsion slots
  // plus restart rebuild/rescore), both O(L)
  auto csort = [&](int *out, int nkeys, auto key) {
    std::vector<int> cnt(nkeys + 1, 0);
    for (int i = 0; i < L; ++i) cnt[nkeys - 1 - key(L0 + i)]++;
    int run = 0;
    for (int k = 0; k < nkeys; ++k) {
      const int t = cnt[k];
      cnt[k] = run;
      run += t;
    }
    for (int i = 0; i < L; ++i) out[cnt[nkeys - 1 - key(L0 + i)]++] = i;
  };
  csort(oa, DS_MAX_ATOMS + 1, [&](int i) { return b->atom_off[i + 1] - b->atom_off[i]; });
  const int kmax = 4096;
  csort(oo, kmax, [&](int i) {
    const int A = b->atom_off[i + 1] - b->atom_off[i], F = b->frag_off[i + 1] - b->frag_off[i];
    return std::min(kmax - 1, ((F + 2) * A) >> 3);
  });
}

void lpt_orders(const ds_batch_desc *b, std::vector<int> &oa, std::vector<int> &oo) {
  oa.resize(b->n_ligands);
  oo.resize(b->n_ligands);
  lpt_orders_range(b, 0, b->n_ligands, oa.data(), oo.data());
}

bool is_pinned(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}


void io_from_buffers(ds_ctx *c) {
  c->io = {(int *)c->b_atom_off.p,    (float4 *)c->b_atoms.p,           (int *)c->b_frag_off.p,
           (uint4 *)c->b_frags.p,     (uint64_t *)c->b_idh.p,           (int *)c->b_order_a.p,
           (int *)c->b_order_o.p,     (ds_result *)c->b_res.p,          (ds_restart_record *)c->b_rrec.p,
           (uint8_t *)c->b_rtors.p,   (float *)c->b_coords.p,           (uint8_t *)c->b_btors.p};
}

// batch-sized device buffers (both families); grows geometrically, never shrinks
int reserve_buffers(ds_ctx *c, int L, int NA, int NF, int N) {
  ++c->gen;  // every caller overwrites (or may reallocate) the per-array buffers
  int rc;
  if ((rc = c->ensure(c->b_atom_off, sizeof(int) * (L + 1))) || (rc = c->ensure(c->b_atoms, 16ull * std::max(NA, 1))) ||
      (rc = c->ensure(c->b_frag_off, sizeof(int) * (L + 1))) || (rc = c->ensure(c->b_frags, 32ull * std::max(NF, 1))) ||
      (rc = c->ensure(c->b_idh, 8ull * L)) || (rc = c->ensure(c->b_order_a, 4ull * L)) ||
      (rc = c->ensure(c->b_order_o, 4ull * L)) || (rc = c->ensure(c->b_keys, 4ull * L * N)) ||
      (rc = c->ensure(c->b_res, sizeof(ds_result) * (size_t)L)) ||
      (rc = c->ensure(c->b_rrec, sizeof(ds_restart_record) * (size_t)L * N)) ||
      (rc = c->ensure(c->b_rtors, (size_t)std::max(NF, 1) * N)) || (rc = c->ensure(c->b_coords, 12ull * std::max(NA, 1))) ||
      (rc = c->ensure(c->b_btors, (size_t)std::max(NF, 1))) || (rc = c->ensure(c->b_queue, 256)))
    return rc;
  io_from_buffers(c);
  return DS_OK;
}

int upload_batch(ds_ctx *c, const ds_batch_desc *b, int N, ds_stats *st) {
  const int L = b->n_ligands;
  const int NA = b->atom_off[L], NF = b->frag_off[L];
  std::vector<int> oa, oo;
  lpt_orders(b, oa, oo);
  int rc;
  if ((rc = reserve_buffers(c, L, NA, NF, N))) return rc;
  // One H2D per array.  Arrays already in pinned memory (ds_host_alloc) are DMA'd directly;
  // pageable ones are first copied into the ctx's pinned staging buffer.
  struct Arr {
    void *dst;
    const void *src;
    size_t bytes;
    bool pinned;
    size_t off;
  } arrs[7] = {{c->b_atom_off.p, b->atom_off, 4ull * (L + 1)},   {c->b_atoms.p, b->atom_xyzt, 16ull * NA},
               {c->b_frag_off.p, b->frag_off, 4ull * (L + 1)},   {c->b_frags.p, b->frag_desc, 32ull * NF},
               {c->b_idh.p, b->id_hash, 8ull * L},               {c->b_order_a.p, oa.data(), 4ull * L},
               {c->b_order_o.p, oo.data(), 4ull * L}};
  size_t o = 0;
  for (int k = 0; k < 7; ++k) {
    arrs[k].pinned = k < 5 && arrs[k].bytes >= (1u << 16) && is_pinned(arrs[k].src);
    arrs[k].off = o;
    if (!arrs[k].pinned) o += (arrs[k].bytes + 255) & ~(size_t)255;
  }
  if ((rc = c->ensure_host(std::max<size_t>(o, 256)))) return rc;
  char *h = (char *)c->h_stage;
  cudaStream_t st_ = c->stream;
  for (int k = 0; k < 7; ++k) {
    if (!arrs[k].bytes) continue;
    const void *src = arrs[k].src;
    if (!arrs[k].pinned) {
      memcpy(h + arrs[k].off, src, arrs[k].bytes);
      src = h + arrs[k].off;
    }
    DS_CUDA(cudaMemcpyAsync(arrs[k].dst, src, arrs[k].bytes, cudaMemcpyHostToDevice, st_));
  }
  if (st) st->h2d_bytes += (int64_t)(4ull * (L + 1) * 2 + 16ull * NA + 32ull * NF + 8ull * L + 8ull * L);
  return DS_OK;
}

// Express path for small calls (the latency family's single ligands): every input array is
// packed into the pinned staging buffer and moved with ONE H2D into an input arena, the kernels
// write their outputs into an output arena that comes back with ONE D2H (each transfer costs a
// PCIe round trip of several microseconds, which dominated the time to result of one ligand).
constexpr size_t kExpressMaxBytes = 4u << 20;

size_t express_in_bytes(const ds_batch_desc *b) {
  const size_t L = (size_t)b->n_ligands, NA = (size_t)b->atom_off[L], NF = (size_t)b->frag_off[L];
  return 2 * 4 * (L + 1) + 16 * NA + 32 * NF + 8 * L + 2 * 4 * L + 7 * 256;
}

// arena sizes for a call of L ligands / NA atoms / NF fragments (256-byte aligned sub-arrays)
void express_sizes(int L, int NA, int NF, int N, size_t *in_bytes, size_t *out_bytes) {
  const size_t sz[7] = {4ull * (L + 1), 16ull * NA, 4ull * (L + 1), 32ull * NF, 8ull * L, 4ull * L, 4ull * L};
  const size_t osz[5] = {sizeof(ds_result) * (size_t)L, sizeof(ds_restart_record) * (size_t)L * N, (size_t)NF * N,
                         12ull * NA, (size_t)NF};
  size_t o = 0;
  for (size_t v : sz) o += (v + 255) & ~(size_t)255;
  *in_bytes = o;
  o = 0;
  for (size_t v : osz) o += (v + 255) & ~(size_t)255;
  *out_bytes = std::max<size_t>(o, 256);
}

int reserve_express(ds_ctx *c, int L, int NA, int NF) {
  size_t ib, ob;
  express_sizes(L, NA, NF, DS_MAX_RESTARTS, &ib, &ob);
  if (ib > kExpressMaxBytes) return DS_OK;  // such calls take the per-array path
  int rc;
  if ((rc = c->ensure(c->x_in, ib)) || (rc = c->ensure(c->x_out, ob)) || (rc = c->ensure_host(ib + ob))) return rc;
  return DS_OK;
}

int upload_express(ds_ctx *c, const ds_batch_desc *b, int N, bool zero_copy_out, ds_stats *st) {
  const int L = b->n_ligands;
  const int NA = b->atom_off[L], NF = b->frag_off[L];
  std::vector<int> oa, oo;
  lpt_orders(b, oa, oo);
  int rc;
  if ((rc = reserve_buffers(c, L, NA, NF, N))) return rc;  // device-only scratch (keys, queue, ...)
  const void *src[7] = {b->atom_off, b->atom_xyzt, b->frag_off, b->frag_desc, b->id_hash, oa.data(), oo.data()};
  const size_t sz[7] = {4ull * (L + 1), 16ull * NA, 4ull * (L + 1), 32ull * NF, 8ull * L, 4ull * L, 4ull * L};
  size_t off[7], o = 0;
  for (int k = 0; k < 7; ++k) {
    off[k] = o;
    o += (sz[k] + 255) & ~(size_t)255;
  }
  const size_t in_bytes = o;
  const size_t osz[5] = {sizeof(ds_result) * (size_t)L, sizeof(ds_restart_record) * (size_t)L * N, (size_t)NF * N,
                         12ull * NA, (size_t)NF};
  o = 0;
  for (int k = 0; k < 5; ++k) {
    c->x_out_off[k] = o;
    o += (osz[k] + 255) & ~(size_t)255;
  }
  const size_t out_bytes = std::max<size_t>(o, 256);
  if ((rc = c->ensure(c->x_in, in_bytes)) || (rc = c->ensure(c->x_out, out_bytes)) ||
      (rc = c->ensure_host(in_bytes + out_bytes)))
    return rc;
  char *h = (char *)c->h_stage;
  for (int k = 0; k < 7; ++k) {
    if (sz[k]) memcpy(h + off[k], src[k], sz[k]);
    const size_t end = k + 1 < 7 ? off[k + 1] : in_bytes;  // alignment padding: defined bytes
    if (end > off[k] + sz[k]) memset(h + off[k] + sz[k], 0, end - off[k] - sz[k]);
  }
  DS_CUDA(cudaMemcpyAsync(c->x_in.p, h, in_bytes, cudaMemcpyHostToDevice, c->stream));
  char *di = (char *)c->x_in.p, *dout = (char *)c->x_out.p;
  c->io.atom_off = (int *)(di + off[0]);
  c->io.atoms = (float4 *)(di + off[1]);
  c->io.frag_off = (int *)(di + off[2]);
  c->io.frags = (uint4 *)(di + off[3]);
  c->io.idh = (uint64_t *)(di + off[4]);
  c->io.order_a = (int *)(di + off[5]);
  c->io.order_o = (int *)(di + off[6]);
  c->io.res = (ds_result *)(dout + c->x_out_off[0]);
  c->io.rrec = (ds_restart_record *)(dout + c->x_out_off[1]);
  c->io.rtors = (uint8_t *)(dout + c->x_out_off[2]);
  c->io.coords = (float *)(dout + c->x_out_off[3]);
  c->io.btors = (uint8_t *)(dout + c->x_out_off[4]);
  c->x_in_bytes = in_bytes;
  c->x_out_bytes = out_bytes;
  c->x_zero_copy = false;
  c->x_rtors_host = nullptr;
  char *hd = nullptr;  // device view of the pinned staging buffer (UVA)
  static const bool zc_env = [] {
    const char *e = getenv("DS_ZERO_COPY");
    return e ? atoi(e) != 0 : true;
  }();
  if (zero_copy_out && zc_env && cudaHostGetDevicePointer((void **)&hd, c->h_stage, 0) == cudaSuccess && hd) {
    hd += in_bytes;
    c->io.res = (ds_result *)(hd + c->x_out_off[0]);
    c->io.rrec = (ds_restart_record *)(hd + c->x_out_off[1]);
    c->io.coords = (float *)(hd + c->x_out_off[3]);
    c->io.btors = (uint8_t *)(hd + c->x_out_off[4]);
    c->x_rtors_host = (uint8_t *)(hd + c->x_out_off[2]);  // rtors itself stays in device memory
    c->x_zero_copy = true;
  } else {
    cudaGetLastError();
  }
  if (st) st->h2d_bytes += (int64_t)in_bytes;
  return DS_OK;
}

int download_express(ds_ctx *c, ds_stats *st) {
  DS_CUDA(cudaMemcpyAsync((char *)c->h_stage + c->x_in_bytes, c->x_out.p, c->x_out_bytes, cudaMemcpyDeviceToHost,
                          c->stream));
  if (st) st->d2h_bytes += (int64_t)c->x_out_bytes;
  return DS_OK;
}

// after the stream has synchronised: scatter the output arena into the caller's buffers
void finish_express(ds_ctx *c, int L, int NA, int NF, int N, const ds_outputs *out) {
  const char *h = (const char *)c->h_stage + c->x_in_bytes;
  if (out->results) memcpy(out->results, h + c->x_out_off[0], sizeof(ds_result) * (size_t)L);
  if (out->restarts) memcpy(out->restarts, h + c->x_out_off[1], sizeof(ds_restart_record) * (size_t)L * N);
  if (out->restart_torsion && NF) memcpy(out->restart_torsion, h + c->x_out_off[2], (size_t)NF * N);
  if (out->best_coords && NA) memcpy(out->best_coords, h + c->x_out_off[3], 12ull * NA);
  if (out->best_torsion && NF) memcpy(out->best_torsion, h + c->x_out_off[4], (size_t)NF);
}

int run_batched_range(ds_ctx *c, const ds_pocket *pk, int L0, int L1, int64_t atom_base, int max_atoms,
                      const DockParams &dp, bool want_coords, bool want_btors, bool want_rrec, ds_stats *st,
                      cudaEvent_t e0, cudaEvent_t e1, cudaEvent_t e2, int *queue);

int run_batched(ds_ctx *c, const ds_pocket *pk, int L, int max_atoms, const DockParams &dp, bool want_coords,
                bool want_btors, bool want_rrec, ds_stats *st) {
  int *queue = (int *)c->b_queue.p;
  DS_CUDA(cudaMemsetAsync(queue, 0, 256, c->stream));
  return run_batched_range(c, pk, 0, L, 0, max_atoms, dp, want_coords, want_btors, want_rrec, st, c->ev[1], c->ev[2],
                           c->ev[3], queue);
}

// Batched family on ligands [L0, L1) of the resident batch (absolute atom/fragment offsets; the
// per-ligand outputs and the order arrays are offset by L0).
int run_batched_range(ds_ctx *c, const ds_pocket *pk, int L0, int L1, int64_t atom_base, int max_atoms,
                      const DockParams &dp_in, bool want_coords, bool want_btors, bool want_rrec, ds_stats *st,
                      cudaEvent_t e0, cudaEvent_t e1, cudaEvent_t e2, int *queue) {
  DockParams dp = dp_in;
  dp.slot_atoms = std::max(1, std::min(max_atoms, DS_MAX_ATOMS));  // select pose-slot stride
  BatchView bt;
  bt.L = L1 - L0;
  bt.atom_off = c->io.atom_off + L0;
  bt.atoms = c->io.atoms;
  bt.frag_off = c->io.frag_off + L0;
  bt.frags = c->io.frags;
  bt.idh = c->io.idh + L0;
  // --- alignment: one CTA per SM, grid staged into smem when it fits ---
  const size_t per_warp = (size_t)align_warp_smem_bytes_host(dp.N);
  const size_t fixed = (size_t)dp.n_a * 16;
#ifndef DS_ALIGN_WARPS
#define DS_ALIGN_WARPS 32
#endif
  int warps_a = DS_ALIGN_WARPS;
  const size_t gb = (size_t)pk->view.grid_bytes;
  int in_smem = gb + fixed + per_warp * 8 <= c->smem_optin;
  if (in_smem) warps_a = (int)std::min<size_t>(DS_ALIGN_WARPS, (c->smem_optin - gb - fixed) / per_warp);
  const size_t smem_a = (in_smem ? gb : 0) + fixed + per_warp * warps_a;
  AlignOut ao{c->sv_keys ? c->sv_keys : (uint32_t *)c->b_keys.p + (size_t)L0 * dp.N};
  cudaEventRecord(e0, c->stream);
  launch_align_batched(pk->view, bt, dp, c->io.order_a + L0, ao, queue, in_smem, c->sm_count, warps_a,
                       smem_a, c->stream);
  cudaEventRecord(e1, c->stream);
  // --- torsion optimisation, then select + rescore: warp per ligand, persistent, occupancy-sized ---
  const int blocks_t = c->sm_count * std::max(1, torsion_blocks_per_sm());
  int rc;
  if (!c->sv_rgv && (rc = c->ensure(c->b_rgv, sizeof(int) * (size_t)dp.N * (size_t)(L1 - L0))))
    return rc;
  OptOut oo = {};
  oo.res = c->io.res + L0;
  oo.rrec = want_rrec ? c->io.rrec + (size_t)L0 * dp.N : nullptr;
  oo.rtors = c->io.rtors;
  oo.final_u = nullptr;
  oo.rgv = c->sv_rgv ? c->sv_rgv : (int *)c->b_rgv.p;
  oo.sel_order = c->sv_sel;
  oo.atom_base = atom_base;
  oo.best_coords = want_coords ? c->io.coords : nullptr;
  oo.best_tors = want_btors ? c->io.btors : nullptr;
  launch_torsion_batched(pk->view, bt, dp, c->io.order_o + L0, ao.keys, oo, queue + 16, blocks_t,
                         c->stream);
  if (e2 == c->ev[3]) cudaEventRecord(c->ev[5], c->stream);  // unchunked: time the select kernel too
  launch_select_batched(pk->view, bt, dp, ao.keys, oo, queue + 32, c->sm_count, c->smem_optin, c->stream);
  cudaEventRecord(e2, c->stream);
  if (st) st->launches += 3;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DS_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
  return DS_OK;
}

// Latency family: alignment spread over (ligand, restart, atom chunk) warps, then one CTA per
// (ligand, restart) for the torsion sweep; the ligand's last CTA selects and rescores.
int run_latency(ds_ctx *c, const ds_pocket *pk, int L, int max_atoms, const DockParams &dp, bool want_coords,
                bool want_btors, bool want_rrec, ds_stats *st) {
  BatchView bt;
  bt.L = L;
  bt.atom_off = c->io.atom_off;
  bt.atoms = c->io.atoms;
  bt.frag_off = c->io.frag_off;
  bt.frags = c->io.frags;
  bt.idh = c->io.idh;
  int rc;
  const size_t nsc = (size_t)L * dp.N * dp.n_rot;
  if ((rc = c->ensure(c->b_lat_scores, 4 * nsc)) || (rc = c->ensure(c->b_lat_recs, latency_rec_bytes() * (size_t)L * dp.N)) ||
      (rc = c->ensure(c->b_lat_done, 4ull * L)) || (rc = c->ensure(c->b_keys, 4ull * L * dp.N)) ||
      (rc = c->ensure(c->b_scratch, sizeof(float4) * (size_t)L * dp.N * DS_MAX_ATOMS)))
    return rc;
  // the kernels leave both buffers zeroed for the next call; clear them only when (re)allocated
  if (c->lat_dirty || c->b_lat_scores.p != c->lat_scores_seen || c->b_lat_done.p != c->lat_done_seen) {
    DS_CUDA(cudaMemsetAsync(c->b_lat_scores.p, 0, c->b_lat_scores.cap, c->stream));
    DS_CUDA(cudaMemsetAsync(c->b_lat_done.p, 0, c->b_lat_done.cap, c->stream));
    c->lat_scores_seen = c->b_lat_scores.p;
    c->lat_done_seen = c->b_lat_done.p;
    c->lat_dirty = false;
  }
  // programmatic dependent launch: the optimisation kernel starts (and stages its shared memory)
  // while the alignment runs; no event between the two kernels then, so align_ms is not split out
  static const bool pdl = [] {
    const char *e = getenv("DS_LATENCY_PDL");
    return e ? atoi(e) != 0 : true;
  }();
  c->lat_pdl = pdl;
  cudaEventRecord(c->ev[1], c->stream);
  OptOut oo = {};
  oo.res = c->io.res;
  oo.rrec = want_rrec ? c->io.rrec : nullptr;
  oo.rtors = c->io.rtors;
  oo.final_u = (float4 *)c->b_scratch.p;
  oo.best_coords = want_coords ? c->io.coords : nullptr;
  oo.best_tors = want_btors ? c->io.btors : nullptr;
  oo.rtors_host = c->x_zero_copy ? c->x_rtors_host : nullptr;
  c->lat_dirty = true;  // until the call has completed (set clean again below / by ds_dock)
  // one ligand over the GPU: the cluster-speculative kernel aligns and optimises in one launch;
  // else the alignment kernel, then the one-CTA-per-restart chain
  if (launch_spread_latency(pk->view, bt, dp, oo, c->b_lat_recs.p, (int *)c->b_lat_done.p, c->stream)) {
    c->lat_pdl = true;  // one kernel: align_ms is not split out
    if (st) {
      st->lat_spread = 10;
      st->launches += 1;
    }
  } else {
    const bool keyed =
        launch_align_latency(pk->view, bt, dp, max_atoms, (int *)c->b_lat_scores.p, (unsigned *)c->b_keys.p, c->stream);
    if (!pdl) cudaEventRecord(c->ev[2], c->stream);
    launch_optimize_latency(pk->view, bt, dp, (int *)c->b_lat_scores.p, keyed ? (const unsigned *)c->b_keys.p : nullptr,
                            oo, c->b_lat_recs.p, (int *)c->b_lat_done.p, pdl, c->stream);
    if (st) {
      st->lat_spread = 1;
      st->launches += 2;
    }
  }
  cudaEventRecord(c->ev[3], c->stream);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DS_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
  return DS_OK;
}

int run_family(ds_ctx *c, const ds_pocket *pk, int family, int L, int NA, int NF, int max_atoms, const DockParams &dp,
               bool want_coords, bool want_btors, bool want_rrec, ds_stats *st) {
  if (family == DS_FAMILY_LATENCY)
    return run_latency(c, pk, L, max_atoms, dp, want_coords, want_btors, want_rrec, st);
  (void)NA;
  (void)NF;
  return run_batched(c, pk, L, max_atoms, dp, want_coords, want_btors, want_rrec, st);
}

int download(ds_ctx *c, int L, int NA, int NF, int N, const ds_outputs *out, ds_stats *st) {
  cudaStream_t s = c->stream;
  if (out->results) {
    DS_CUDA(cudaMemcpyAsync(out->results, c->b_res.p, sizeof(ds_result) * (size_t)L, cudaMemcpyDeviceToHost, s));
    if (st) st->d2h_bytes += sizeof(ds_result) * (int64_t)L;
  }
  if (out->best_coords && NA) {
    DS_CUDA(cudaMemcpyAsync(out->best_coords, c->b_coords.p, 12ull * NA, cudaMemcpyDeviceToHost, s));
    if (st) st->d2h_bytes += 12ll * NA;
  }
  if (out->best_torsion && NF) {
    DS_CUDA(cudaMemcpyAsync(out->best_torsion, c->b_btors.p, (size_t)NF, cudaMemcpyDeviceToHost, s));
    if (st) st->d2h_bytes += NF;
  }
  if (out->restarts) {
    DS_CUDA(cudaMemcpyAsync(out->restarts, c->b_rrec.p, sizeof(ds_restart_record) * (size_t)L * N, cudaMemcpyDeviceToHost, s));
    if (st) st->d2h_bytes += (int64_t)sizeof(ds_restart_record) * L * N;
  }
  if (out->restart_torsion && NF) {
    DS_CUDA(cudaMemcpyAsync(out->restart_torsion, c->b_rtors.p, (size_t)NF * N, cudaMemcpyDeviceToHost, s));
    if (st) st->d2h_bytes += (int64_t)NF * N;
  }
  return DS_OK;
}

void fill_times(ds_ctx *c, ds_stats *st, bool with_copies, bool family_batched) {
  if (!st) return;
  float t = 0.f;
  if (!family_batched && c->lat_pdl) {  // overlapped kernels: both in optimize_ms
    st->align_ms = 0.f;
    cudaEventElapsedTime(&t, c->ev[1], c->ev[3]);
    st->optimize_ms = t;
  } else {
    cudaEventElapsedTime(&t, c->ev[1], c->ev[2]);
    st->align_ms = t;
    cudaEventElapsedTime(&t, c->ev[2], c->ev[3]);
    st->optimize_ms = t;
  }
  st->select_ms = 0.f;
  if (family_batched && cudaEventElapsedTime(&t, c->ev[5], c->ev[3]) == cudaSuccess) st->select_ms = t;
  cudaEventElapsedTime(&t, with_copies ? c->ev[0] : c->ev[1], with_copies ? c->ev[4] : c->ev[3]);
  st->total_ms = t;
}

// Large batched calls: the batch is split into nch contiguous chunks; chunk k's H2D on the copy
// stream overlaps chunk k-1's kernels, and chunk k's D2H overlaps chunk k+1's kernels.
int dock_pipelined(ds_ctx *c, const ds_pocket *pk, const ds_batch_desc *b, const DockParams &dp,
                   const ds_outputs *out, ds_stats *st, int nch) {
  const int L = b->n_ligands, N = dp.N;
  const int NA = b->atom_off[L], NF = b->frag_off[L];
  int rc;
  if ((rc = reserve_buffers(c, L, NA, NF, N)) || (rc = c->ensure(c->b_queue, 256ull * nch))) return rc;
  while ((int)c->pev.size() < 4 * nch) {
    cudaEvent_t e;
    DS_CUDA(cudaEventCreate(&e));
    c->pev.push_back(e);
  }
  std::vector<int> bounds(nch + 1);
  // tapered chunks: the first and last are a quarter of the inner ones, so the un-overlapped head
  // (first H2D) and tail (last D2H) of the pipeline stay short (DS_PIPELINE_TAPER = the end-chunk
  // weight; 0 or >= 1: equal chunks)
  {
    const char *e = getenv("DS_PIPELINE_TAPER");
    const double tw = e ? atof(e) : 0.25;
    const bool taper = tw > 0.0 && tw < 1.0 && nch >= 3;
    std::vector<double> w(nch, 1.0);
    if (taper) w[0] = w[nch - 1] = tw;
    double tot = 0, run = 0;
    for (double x : w) tot += x;
    bounds[0] = 0;
    for (int k = 0; k < nch; ++k) {
      run += w[k];
      bounds[k + 1] = k + 1 == nch ? L : (int)((double)L * run / tot);
    }
  }
  // host side: LPT orders per chunk; pageable inputs go through the pinned staging buffer
  struct Src {
    const void *p;
    size_t bytes;
  } src[5] = {{b->atom_off, 4ull * (L + 1)}, {b->frag_off, 4ull * (L + 1)}, {b->id_hash, 8ull * L},
              {b->atom_xyzt, 16ull * NA}, {b->frag_desc, 32ull * NF}};
  size_t off[7], o = 0;
  bool pinned[5];
  for (int k = 0; k < 5; ++k) {
    pinned[k] = src[k].bytes >= (1u << 16) && is_pinned(src[k].p);
    off[k] = o;
    if (!pinned[k]) o += (src[k].bytes + 255) & ~(size_t)255;
  }
  off[5] = o;
  o += (4ull * L + 255) & ~(size_t)255;
  off[6] = o;
  o += (4ull * L + 255) & ~(size_t)255;
  if ((rc = c->ensure_host(o))) return rc;
  char *h = (char *)c->h_stage;
  const char *hp[5];
  for (int k = 0; k < 5; ++k) {
    hp[k] = (const char *)src[k].p;
    if (!pinned[k] && src[k].bytes) {
      memcpy(h + off[k], src[k].p, src[k].bytes);
      hp[k] = h + off[k];
    }
  }
  int *oa = (int *)(h + off[5]), *oo = (int *)(h + off[6]);
  cudaStream_t cs = c->copy;
  cudaEventRecord(c->ev[0], cs);
  DS_CUDA(cudaMemcpyAsync(c->b_atom_off.p, hp[0], src[0].bytes, cudaMemcpyHostToDevice, cs));
  DS_CUDA(cudaMemcpyAsync(c->b_frag_off.p, hp[1], src[1].bytes, cudaMemcpyHostToDevice, cs));
  DS_CUDA(cudaMemcpyAsync(c->b_idh.p, hp[2], src[2].bytes, cudaMemcpyHostToDevice, cs));
  int *queue = (int *)c->b_queue.p;
  DS_CUDA(cudaMemsetAsync(queue, 0, 256ull * nch, c->stream));
  // D2H of chunk j on the copy stream, after its kernels
  auto d2h = [&](int j) -> int {
    const int L0 = bounds[j], L1 = bounds[j + 1];
    DS_CUDA(cudaStreamWaitEvent(cs, c->pev[4 * j + 3], 0));
    const size_t a0 = b->atom_off[L0], a1 = b->atom_off[L1], f0 = b->frag_off[L0], f1 = b->frag_off[L1];
    DS_CUDA(cudaMemcpyAsync(out->results + L0, (ds_result *)c->b_res.p + L0, sizeof(ds_result) * (L1 - L0),
                            cudaMemcpyDeviceToHost, cs));
    if (out->best_coords && a1 > a0)
      DS_CUDA(cudaMemcpyAsync(out->best_coords + 3 * a0, (float *)c->b_coords.p + 3 * a0, 12 * (a1 - a0),
                              cudaMemcpyDeviceToHost, cs));
    if (out->best_torsion && f1 > f0)
      DS_CUDA(cudaMemcpyAsync(out->best_torsion + f0, (uint8_t *)c->b_btors.p + f0, f1 - f0, cudaMemcpyDeviceToHost, cs));
    if (out->restarts)
      DS_CUDA(cudaMemcpyAsync(out->restarts + (size_t)L0 * N, (ds_restart_record *)c->b_rrec.p + (size_t)L0 * N,
                              sizeof(ds_restart_record) * (size_t)(L1 - L0) * N, cudaMemcpyDeviceToHost, cs));
    if (out->restart_torsion && f1 > f0)
      DS_CUDA(cudaMemcpyAsync(out->restart_torsion + f0 * N, (uint8_t *)c->b_rtors.p + f0 * N, (f1 - f0) * N,
                              cudaMemcpyDeviceToHost, cs));
    if (st)
      st->d2h_bytes += (int64_t)(sizeof(ds_result) * (L1 - L0) + (out->best_coords ? 12 * (a1 - a0) : 0) +
                                 (out->best_torsion ? f1 - f0 : 0) +
                                 (out->restarts ? sizeof(ds_restart_record) * (size_t)(L1 - L0) * N : 0) +
                                 (out->restart_torsion ? (f1 - f0) * N : 0));
    return DS_OK;
  };
  // copy stream order: H2D(0), H2D(1), D2H(0), H2D(2), D2H(1), ...: every H2D is queued before the
  // D2H that waits on the previous chunk's kernels, so uploads run ahead of the compute stream
  for (int k = 0; k < nch; ++k) {
    const int L0 = bounds[k], L1 = bounds[k + 1];
    // chunk k's LPT orders are computed on the host while the device works on chunk k-1
    lpt_orders_range(b, L0, L1, oa + L0, oo + L0);
    const size_t a0 = b->atom_off[L0], a1 = b->atom_off[L1], f0 = b->frag_off[L0], f1 = b->frag_off[L1];
    DS_CUDA(cudaMemcpyAsync((float4 *)c->b_atoms.p + a0, hp[3] + 16 * a0, 16 * (a1 - a0), cudaMemcpyHostToDevice, cs));
    if (f1 > f0)
      DS_CUDA(cudaMemcpyAsync((char *)c->b_frags.p + 32 * f0, hp[4] + 32 * f0, 32 * (f1 - f0), cudaMemcpyHostToDevice, cs));
    DS_CUDA(cudaMemcpyAsync((int *)c->b_order_a.p + L0, oa + L0, 4ull * (L1 - L0), cudaMemcpyHostToDevice, cs));
    DS_CUDA(cudaMemcpyAsync((int *)c->b_order_o.p + L0, oo + L0, 4ull * (L1 - L0), cudaMemcpyHostToDevice, cs));
    cudaEventRecord(c->pev[4 * k], cs);
    DS_CUDA(cudaStreamWaitEvent(c->stream, c->pev[4 * k], 0));
    int amax = 1;
    for (int i = L0; i < L1; ++i) amax = std::max(amax, b->atom_off[i + 1] - b->atom_off[i]);
    if ((rc = run_batched_range(c, pk, L0, L1, b->atom_off[L0], amax, dp,
                                out->best_coords != nullptr, out->best_torsion != nullptr, out->restarts != nullptr,
                                st, c->pev[4 * k + 1], c->pev[4 * k + 2], c->pev[4 * k + 3], queue + 64 * k)))
      return rc;
    if (k > 0 && (rc = d2h(k - 1))) return rc;
  }
  if ((rc = d2h(nch - 1))) return rc;
  if (st) st->h2d_bytes += (int64_t)(src[0].bytes + src[1].bytes + src[2].bytes + src[3].bytes + src[4].bytes + 8ull * L);
  cudaEventRecord(c->ev[4], cs);
  DS_CUDA(cudaStreamSynchronize(cs));
  DS_CUDA(cudaStreamSynchronize(c->stream));
  if (st) {
    float t = 0.f;
    st->align_ms = st->optimize_ms = 0.f;
    for (int k = 0; k < nch; ++k) {
      cudaEventElapsedTime(&t, c->pev[4 * k + 1], c->pev[4 * k + 2]);
      st->align_ms += t;
      cudaEventElapsedTime(&t, c->pev[4 * k + 2], c->pev[4 * k + 3]);
      st->optimize_ms += t;
    }
    cudaEventElapsedTime(&t, c->ev[0], c->ev[4]);
    st->total_ms = t;
  }
  return DS_OK;
}

int pipeline_chunks(int L) {
  const char *e = getenv("DS_PIPELINE_CHUNKS");
  int n = e ? atoi(e) : 4;  // measured best of {1, 2, 4, 8} on the 200k-ligand bench step
  if (n < 1) n = 1;
  if (L < 20000) return 1;
  return std::min(n, L / 5000);
}

}  // namespace

extern "C" {

int ds_dock(ds_ctx *c, const ds_pocket *pk, const ds_batch_desc *b, const ds_dock_config *cfg, int family,
            const ds_outputs *out, ds_stats *st) {
  if (!c || !pk || !out || !out->results) return fail(DS_ERR_INVALID_ARG, "NULL argument");
  if (family != DS_FAMILY_BATCHED && family != DS_FAMILY_LATENCY) return fail(DS_ERR_INVALID_ARG, "unknown family %d", family);
  DockParams dp;
  int rc;
  if ((rc = check_config(cfg, pk, &dp)) || (rc = check_batch(b))) return rc;
  if (st) memset(st, 0, sizeof *st);
  const int L = b->n_ligands;
  if (L == 0) return DS_OK;
  DS_CUDA(enter_device(c->device));
  if (family == DS_FAMILY_BATCHED) {
    const int nch = pipeline_chunks(L);
    if (nch > 1) return dock_pipelined(c, pk, b, dp, out, st, nch);
  }
  const int NA = b->atom_off[L], NF = b->frag_off[L];
  const bool express = express_in_bytes(b) <= kExpressMaxBytes;
  cudaEventRecord(c->ev[0], c->stream);
  c->x_zero_copy = false;
  if ((rc = express ? upload_express(c, b, dp.N, family == DS_FAMILY_LATENCY, st) : upload_batch(c, b, dp.N, st)))
    return rc;
  int max_atoms = 0;
  for (int i = 0; i < L; ++i) max_atoms = std::max(max_atoms, b->atom_off[i + 1] - b->atom_off[i]);
  if ((rc = run_family(c, pk, family, L, NA, NF, max_atoms, dp, out->best_coords != nullptr,
                       out->best_torsion != nullptr, out->restarts != nullptr, st)))
    return rc;
  if (express && c->x_zero_copy) {
    if (st) st->d2h_bytes += (int64_t)c->x_out_bytes;  // written by the kernels over the bus instead
  } else if ((rc = express ? download_express(c, st) : download(c, L, NA, NF, dp.N, out, st))) {
    return rc;
  }
  c->x_zero_copy = false;
  cudaEventRecord(c->ev[4], c->stream);
  DS_CUDA(cudaStreamSynchronize(c->stream));
  if (family == DS_FAMILY_LATENCY) c->lat_dirty = false;  // a completed call leaves its scratch zeroed
  if (express) finish_express(c, L, NA, NF, dp.N, out);
  fill_times(c, st, true, family == DS_FAMILY_BATCHED);
  return DS_OK;
}

int ds_ctx_reserve(ds_ctx *c, int max_ligands, int max_atoms, int max_frags, const ds_dock_config *cfg) {
  if (!c || !cfg || max_ligands < 1 || max_atoms < 1 || max_frags < 0) return fail(DS_ERR_INVALID_ARG, "bad argument");
  if (cfg->restarts_n < 1 || cfg->restarts_n > DS_MAX_RESTARTS || cfg->alignment_step_deg < 1 ||
      360 % cfg->alignment_step_deg)
    return fail(DS_ERR_INVALID_ARG, "bad config");
  DS_CUDA(enter_device(c->device));
  const int N = cfg->restarts_n, na = 360 / cfg->alignment_step_deg;
  const size_t L = (size_t)max_ligands;
  int rc;
  if ((rc = reserve_buffers(c, max_ligands, max_atoms, max_frags, DS_MAX_RESTARTS)) ||
      (rc = c->ensure(c->b_lat_scores, 4 * L * N * na * na)) ||
      (rc = c->ensure(c->b_lat_recs, latency_rec_bytes() * L * N)) || (rc = c->ensure(c->b_lat_done, 4 * L)) ||
      (rc = c->ensure(c->b_scratch, sizeof(float4) * std::max(L * DS_MAX_ATOMS, (size_t)max_atoms) * N)) ||
      (rc = c->ensure(c->b_rgv, sizeof(int) * L * N)) ||
      (rc = reserve_express(c, max_ligands, max_atoms, max_frags)) ||
      (rc = c->ensure_host((size_t)max_atoms * 16 + (size_t)max_frags * 32 + L * 32 + 4096)))
    return rc;
  return DS_OK;
}

int ds_batch_upload(ds_ctx *c, const ds_batch_desc *b, ds_dev_batch **out) {
  if (!c || !out) return fail(DS_ERR_INVALID_ARG, "NULL argument");
  int rc;
  if ((rc = check_batch(b))) return rc;
  DS_CUDA(enter_device(c->device));
  ds_dev_batch *d = new ds_dev_batch();
  d->ctx = c;
  d->L = b->n_ligands;
  d->atom_off.assign(b->atom_off, b->atom_off + d->L + 1);
  d->frag_off.assign(b->frag_off, b->frag_off + d->L + 1);
  d->n_atoms = b->atom_off[d->L];
  d->n_frags = b->frag_off[d->L];
  if ((rc = upload_batch(c, b, DS_MAX_RESTARTS, nullptr))) {
    delete d;
    return rc;
  }
  d->gen = c->gen;
  DS_CUDA(cudaStreamSynchronize(c->stream));
  *out = d;
  return DS_OK;
}

static int stale(const ds_ctx *c, const ds_dev_batch *d) {
  return fail(DS_ERR_INVALID_ARG,
              "stale resident batch: ctx %p reused its buffers (generation %llu, batch %llu) for a later "
              "upload / generation / ds_dock / op call", (const void *)c, (unsigned long long)c->gen,
              (unsigned long long)d->gen);
}

int ds_dock_resident(ds_ctx *c, const ds_pocket *pk, ds_dev_batch *d, const ds_dock_config *cfg, int family,
                     ds_stats *st) {
  if (!c || !pk || !d || d->ctx != c) return fail(DS_ERR_INVALID_ARG, "bad argument");
  if (d->gen != c->gen) return stale(c, d);
  DockParams dp;
  int rc;
  if ((rc = check_config(cfg, pk, &dp))) return rc;
  if (st) memset(st, 0, sizeof *st);
  if (d->L == 0) {  // nothing to dock; the (empty) download is still valid
    d->N = dp.N;
    d->docked = true;
    return DS_OK;
  }
  DS_CUDA(enter_device(c->device));
  int max_atoms = 0;
  for (int i = 0; i < d->L; ++i) max_atoms = std::max(max_atoms, d->atom_off[i + 1] - d->atom_off[i]);
  io_from_buffers(c);  // the resident batch lives in the per-array buffers (not an express arena)
  c->x_zero_copy = false;
  if ((rc = run_family(c, pk, family, d->L, d->n_atoms, d->n_frags, max_atoms, dp, true, true, true, st))) return rc;
  DS_CUDA(cudaStreamSynchronize(c->stream));
  if (family == DS_FAMILY_LATENCY) c->lat_dirty = false;
  d->N = dp.N;
  d->docked = true;
  fill_times(c, st, false, family == DS_FAMILY_BATCHED);
  return DS_OK;
}

int ds_batch_download(ds_ctx *c, ds_dev_batch *d, const ds_outputs *out) {
  if (!c || !d || !out || d->ctx != c) return fail(DS_ERR_INVALID_ARG, "bad argument");
  if (d->gen != c->gen) return stale(c, d);
  if (!d->docked) return fail(DS_ERR_INVALID_ARG, "batch has not been docked");
  if (d->L == 0) return DS_OK;
  int rc;
  if ((rc = download(c, d->L, d->n_atoms, d->n_frags, d->N, out, nullptr))) return rc;
  DS_CUDA(cudaStreamSynchronize(c->stream));
  return DS_OK;
}

void ds_batch_destroy(ds_dev_batch *d) { delete d; }

// ---- engine stream (batched_engine.run) ---------------------------------------
// The whole packed ligand stream of one engine run lives on the device: producers upload the
// ranges they have packed, each batch the bucketizer detaches is docked as a list of stream ligand
// numbers (the kernels take queue item -> ligand orders), outputs stay at the stream's ligand /
// atom / fragment offsets and come back with one download — no per-batch gather, H2D, D2H or
// scatter on the host.  Buffers grow geometrically and are kept across runs.
}  // extern "C"

struct ds_stream {
  int device = 0;
  int L = 0, NA = 0, NF = 0, N = 0;
  std::vector<int> atom_off, frag_off;  // host copies: LPT keys and the batch's largest ligand
  DevBuf atom_off_d, atoms, frag_off_d, frags, idh, keys, rgv, res, rtors, coords, btors;
  int64_t allocs = 0;
  int grow(DevBuf &b, size_t bytes) {
    bytes = std::max<size_t>(bytes, 256);
    if (bytes <= b.cap) return DS_OK;
    size_t nc = std::max(bytes, b.cap * 3 / 2);
    nc = (nc + 255) & ~(size_t)255;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
    cudaError_t e = cudaMalloc(&b.p, nc);
    if (e != cudaSuccess) return fail(DS_ERR_OOM, "cudaMalloc(%zu): %s", nc, cudaGetErrorString(e));
    b.cap = nc;
    ++allocs;
    return DS_OK;
  }
  ~ds_stream() {
    cudaSetDevice(device);
    for (DevBuf *b : {&atom_off_d, &atoms, &frag_off_d, &frags, &idh, &keys, &rgv, &res, &rtors, &coords, &btors})
      if (b->p) cudaFree(b->p);
  }
};

extern "C" {

int ds_stream_create(ds_ctx *c, ds_stream **out) {
  if (!c || !out) return fail(DS_ERR_INVALID_ARG, "NULL argument");
  *out = new ds_stream();
  (*out)->device = c->device;
  return DS_OK;
}

void ds_stream_destroy(ds_stream *s) { delete s; }

int ds_stream_begin(ds_stream *s, int32_t n_ligands, const int32_t *atom_off, const int32_t *frag_off,
                    int32_t restarts) {
  if (!s || n_ligands < 0 || (n_ligands > 0 && (!atom_off || !frag_off)) || restarts < 1 ||
      restarts > DS_MAX_RESTARTS)
    return fail(DS_ERR_INVALID_ARG, "bad argument");
  const int L = n_ligands;
  const int NA = L ? atom_off[L] : 0, NF = L ? frag_off[L] : 0;
  if (L && (atom_off[0] != 0 || frag_off[0] != 0)) return fail(DS_ERR_INVALID_ARG, "offsets must start at 0");
  for (int i = 0; i < L; ++i) {
    const int A = atom_off[i + 1] - atom_off[i];
    if (A < 1 || A > DS_MAX_ATOMS) return fail(DS_ERR_TOO_MANY_ATOMS, "ligand %d has %d atoms", i, A);
    if (frag_off[i + 1] < frag_off[i]) return fail(DS_ERR_INVALID_ARG, "frag_off not monotone");
  }
  DS_CUDA(enter_device(s->device));
  int rc;
  if ((rc = s->grow(s->atom_off_d, 4ull * (L + 1))) || (rc = s->grow(s->atoms, 16ull * NA)) ||
      (rc = s->grow(s->frag_off_d, 4ull * (L + 1))) || (rc = s->grow(s->frags, 32ull * NF)) ||
      (rc = s->grow(s->idh, 8ull * L)) || (rc = s->grow(s->keys, 4ull * L * restarts)) ||
      (rc = s->grow(s->rgv, 4ull * L * restarts)) || (rc = s->grow(s->res, sizeof(ds_result) * (size_t)L)) ||
      (rc = s->grow(s->rtors, (size_t)NF * restarts)) || (rc = s->grow(s->coords, 12ull * NA)) ||
      (rc = s->grow(s->btors, (size_t)NF)))
    return rc;
  s->L = L;
  s->NA = NA;
  s->NF = NF;
  s->N = restarts;
  s->atom_off.assign(atom_off, atom_off + L + 1);
  s->frag_off.assign(frag_off, frag_off + L + 1);
  if (!L) {
    s->atom_off.assign(1, 0);
    s->frag_off.assign(1, 0);
  }
  // records of ligands no batch docks (invalid ones) read back as zeros
  DS_CUDA(cudaMemcpy(s->atom_off_d.p, s->atom_off.data(), 4ull * (L + 1), cudaMemcpyHostToDevice));
  DS_CUDA(cudaMemcpy(s->frag_off_d.p, s->frag_off.data(), 4ull * (L + 1), cudaMemcpyHostToDevice));
  DS_CUDA(cudaMemset(s->res.p, 0, sizeof(ds_result) * (size_t)std::max(L, 1)));
  return DS_OK;
}

int ds_stream_upload(ds_stream *s, int32_t lo, int32_t hi, const float *atom_xyzt, const uint32_t *frag_desc,
                     const uint64_t *id_hash) {
  if (!s || lo < 0 || hi < lo || hi > s->L || !atom_xyzt || !id_hash || (!frag_desc && s->NF))
    return fail(DS_ERR_INVALID_ARG, "bad argument");
  if (lo == hi) return DS_OK;
  DS_CUDA(enter_device(s->device));
  // the calling thread's own stream: producers upload disjoint ranges concurrently
  cudaStream_t st = cudaStreamPerThread;
  const size_t a0 = s->atom_off[lo], a1 = s->atom_off[hi], f0 = s->frag_off[lo], f1 = s->frag_off[hi];
  DS_CUDA(cudaMemcpyAsync((float4 *)s->atoms.p + a0, atom_xyzt + 4 * a0, 16 * (a1 - a0), cudaMemcpyHostToDevice, st));
  if (f1 > f0)
    DS_CUDA(cudaMemcpyAsync((char *)s->frags.p + 32 * f0, (const char *)frag_desc + 32 * f0, 32 * (f1 - f0),
                            cudaMemcpyHostToDevice, st));
  DS_CUDA(cudaMemcpyAsync((uint64_t *)s->idh.p + lo, id_hash + lo, 8ull * (hi - lo), cudaMemcpyHostToDevice, st));
  DS_CUDA(cudaStreamSynchronize(st));
  return DS_OK;
}

int ds_stream_dock(ds_ctx *c, const ds_pocket *pk, ds_stream *s, const int32_t *sel, int32_t n_sel,
                   const ds_dock_config *cfg, ds_stats *st) {
  if (!c || !pk || !s || !cfg || n_sel < 0 || (n_sel && !sel)) return fail(DS_ERR_INVALID_ARG, "bad argument");
  if (c->device != s->device) return fail(DS_ERR_INVALID_ARG, "stream and context on different devices");
  DockParams dp;
  int rc;
  if ((rc = check_config(cfg, pk, &dp))) return rc;
  if (dp.N != s->N) return fail(DS_ERR_INVALID_ARG, "restarts %d != the stream's %d", dp.N, s->N);
  if (st) memset(st, 0, sizeof *st);
  if (!n_sel) return DS_OK;
  // LPT orders of the batch (stream ligand numbers): alignment ~ A, optimisation ~ (F + 2) * A,
  // descending, stable counting sorts
  int max_atoms = 0;
  for (int k = 0; k < n_sel; ++k) {
    const int i = sel[k];
    if (i < 0 || i >= s->L) return fail(DS_ERR_INVALID_ARG, "ligand %d outside the stream", i);
    max_atoms = std::max(max_atoms, s->atom_off[i + 1] - s->atom_off[i]);
  }
  DS_CUDA(enter_device(c->device));
  if ((rc = c->ensure(c->b_order_a, 4ull * n_sel)) || (rc = c->ensure(c->b_order_o, 4ull * n_sel)) ||
      (rc = c->ensure(c->b_queue, 256)) || (rc = c->ensure_host(8ull * n_sel)))
    return rc;
  int *oa = (int *)c->h_stage, *oo = oa + n_sel;
  auto csort = [&](int *out, int nkeys, auto key) {
    std::vector<int> cnt(nkeys + 1, 0);
    for (int k = 0; k < n_sel; ++k) cnt[nkeys - 1 - key(sel[k])]++;
    int run = 0;
    for (int q = 0; q < nkeys; ++q) {
      const int t = cnt[q];
      cnt[q] = run;
      run += t;
    }
    for (int k = 0; k < n_sel; ++k) out[cnt[nkeys - 1 - key(sel[k])]++] = sel[k];
  };
  const int *ao = s->atom_off.data(), *fo = s->frag_off.data();
  csort(oa, DS_MAX_ATOMS + 1, [&](int i) { return ao[i + 1] - ao[i]; });
  csort(oo, 4096, [&](int i) { return std::min(4095, ((fo[i + 1] - fo[i] + 2) * (ao[i + 1] - ao[i])) >> 3); });
  cudaEventRecord(c->ev[0], c->stream);
  DS_CUDA(cudaMemcpyAsync(c->b_order_a.p, oa, 4ull * n_sel, cudaMemcpyHostToDevice, c->stream));
  DS_CUDA(cudaMemcpyAsync(c->b_order_o.p, oo, 4ull * n_sel, cudaMemcpyHostToDevice, c->stream));
  DS_CUDA(cudaMemsetAsync(c->b_queue.p, 0, 256, c->stream));
  c->io = {(int *)s->atom_off_d.p, (float4 *)s->atoms.p, (int *)s->frag_off_d.p, (uint4 *)s->frags.p,
           (uint64_t *)s->idh.p,   (int *)c->b_order_a.p, (int *)c->b_order_o.p, (ds_result *)s->res.p,
           nullptr,               (uint8_t *)s->rtors.p, (float *)s->coords.p,  (uint8_t *)s->btors.p};
  c->x_zero_copy = false;
  c->sv_keys = (uint32_t *)s->keys.p;
  c->sv_rgv = (int *)s->rgv.p;
  c->sv_sel = (const int *)c->b_order_o.p;
  ++c->gen;  // the per-array views no longer describe a resident batch
  rc = run_batched_range(c, pk, 0, n_sel, 0, max_atoms, dp, true, true, false, st, c->ev[1], c->ev[2], c->ev[3],
                         (int *)c->b_queue.p);
  c->sv_keys = nullptr;
  c->sv_rgv = nullptr;
  c->sv_sel = nullptr;
  io_from_buffers(c);
  if (rc) return rc;
  cudaEventRecord(c->ev[4], c->stream);
  DS_CUDA(cudaStreamSynchronize(c->stream));
  fill_times(c, st, false, true);
  if (st) st->h2d_bytes = 8ll * n_sel;
  return DS_OK;
}

int ds_stream_download(ds_ctx *c, ds_stream *s, const ds_outputs *out) {
  if (!c || !s || !out || out->restarts || out->restart_torsion) return fail(DS_ERR_INVALID_ARG, "bad argument");
  if (c->device != s->device) return fail(DS_ERR_INVALID_ARG, "stream and context on different devices");
  if (!s->L) return DS_OK;
  DS_CUDA(enter_device(c->device));
  if (out->results)
    DS_CUDA(cudaMemcpyAsync(out->results, s->res.p, sizeof(ds_result) * (size_t)s->L, cudaMemcpyDeviceToHost,
                            c->stream));
  if (out->best_coords && s->NA)
    DS_CUDA(cudaMemcpyAsync(out->best_coords, s->coords.p, 12ull * s->NA, cudaMemcpyDeviceToHost, c->stream));
  if (out->best_torsion && s->NF)
    DS_CUDA(cudaMemcpyAsync(out->best_torsion, s->btors.p, (size_t)s->NF, cudaMemcpyDeviceToHost, c->stream));
  DS_CUDA(cudaStreamSynchronize(c->stream));
  return DS_OK;
}

int ds_generate_resident(ds_ctx *c, int64_t seed, int64_t first_index, int32_t count, const int32_t *shapes,
                         ds_dev_batch **out, float *device_ms) {
  if (!c || !out || !shapes || count < 0) return fail(DS_ERR_INVALID_ARG, "bad argument");
  // offsets on the host (hydrogen counts only: ~20 ns per ligand), InfeasibleShape checked there
  std::vector<int32_t> ao((size_t)count + 1), bo((size_t)count + 1), fo((size_t)count + 1);
  int rc = ds_generate_ligands(seed, first_index, count, shapes, ao.data(), bo.data(), fo.data(), nullptr, nullptr,
                               nullptr, nullptr, nullptr);
  if (rc == DS_ERR_INFEASIBLE_SHAPE) return fail(rc, "InfeasibleShape: fragments >= heavy - 1 or atoms out of range");
  if (rc) return fail(rc, "bad generator arguments");
  const int L = count, NA = ao[L], NF = fo[L];
  DS_CUDA(enter_device(c->device));
  ds_batch_desc b;
  memset(&b, 0, sizeof b);
  b.n_ligands = L;
  b.atom_off = ao.data();
  b.frag_off = fo.data();
  std::vector<int> oa, oo;
  lpt_orders(&b, oa, oo);
  if ((rc = reserve_buffers(c, L, NA, NF, DS_MAX_RESTARTS)) || (rc = c->ensure_host(16ull * L + 64))) return rc;
  // the shapes ride in the key buffer (8 B per ligand <= 4 N B; the alignment kernel overwrites it)
  int *d_shapes = (int *)c->b_keys.p;
  char *h = (char *)c->h_stage;
  memcpy(h, shapes, 8ull * L);
  cudaStream_t st = c->stream;
  cudaEventRecord(c->ev[0], st);
  DS_CUDA(cudaMemcpyAsync(d_shapes, h, 8ull * L, cudaMemcpyHostToDevice, st));
  DS_CUDA(cudaMemcpyAsync(c->b_atom_off.p, ao.data(), 4ull * (L + 1), cudaMemcpyHostToDevice, st));
  DS_CUDA(cudaMemcpyAsync(c->b_frag_off.p, fo.data(), 4ull * (L + 1), cudaMemcpyHostToDevice, st));
  DS_CUDA(cudaMemcpyAsync(c->b_order_a.p, oa.data(), 4ull * L, cudaMemcpyHostToDevice, st));
  DS_CUDA(cudaMemcpyAsync(c->b_order_o.p, oo.data(), 4ull * L, cudaMemcpyHostToDevice, st));
  cudaEventRecord(c->ev[1], st);
  launch_generate_ligands(seed, first_index, L, d_shapes, (const int *)c->b_atom_off.p, (const int *)c->b_frag_off.p,
                          (float4 *)c->b_atoms.p, (uint32_t *)c->b_frags.p, (uint64_t *)c->b_idh.p, c->sm_count, st);
  cudaEventRecord(c->ev[2], st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(DS_ERR_CUDA, "generator launch: %s", cudaGetErrorString(e));
  DS_CUDA(cudaStreamSynchronize(st));
  if (device_ms) cudaEventElapsedTime(device_ms, c->ev[1], c->ev[2]);
  ds_dev_batch *d = new ds_dev_batch();
  d->ctx = c;
  d->gen = c->gen;
  d->L = L;
  d->atom_off.assign(ao.begin(), ao.end());
  d->frag_off.assign(fo.begin(), fo.end());
  d->n_atoms = NA;
  d->n_frags = NF;
  *out = d;
  return DS_OK;
}

int ds_batch_read_inputs(ds_ctx *c, const ds_dev_batch *d, float *atom_xyzt, uint32_t *frag_desc, uint64_t *id_hash) {
  if (!c || !d || d->ctx != c) return fail(DS_ERR_INVALID_ARG, "bad argument");
  if (d->gen != c->gen) return stale(c, d);
  DS_CUDA(enter_device(c->device));
  if (atom_xyzt && d->n_atoms)
    DS_CUDA(cudaMemcpyAsync(atom_xyzt, c->b_atoms.p, 16ull * d->n_atoms, cudaMemcpyDeviceToHost, c->stream));
  if (frag_desc && d->n_frags)
    DS_CUDA(cudaMemcpyAsync(frag_desc, c->b_frags.p, 32ull * d->n_frags, cudaMemcpyDeviceToHost, c->stream));
  if (id_hash && d->L) DS_CUDA(cudaMemcpyAsync(id_hash, c->b_idh.p, 8ull * d->L, cudaMemcpyDeviceToHost, c->stream));
  DS_CUDA(cudaStreamSynchronize(c->stream));
  return DS_OK;
}

int ds_build_pocket_grid_device(ds_ctx *c, const float *atom_xyz, int32_t n_atoms, float spacing, float padding,
                                float origin[3], int32_t dims[3], int32_t *values, float *device_ms) {
  if (!c || !values) return fail(DS_ERR_INVALID_ARG, "NULL argument");
  int rc = ds_build_pocket_grid(atom_xyz, n_atoms, spacing, padding, origin, dims, nullptr);  // origin, dims
  if (rc == DS_ERR_EMPTY_POCKET) return fail(rc, "build_pocket needs at least one atom");
  if (rc) return fail(rc, "bad build_pocket arguments");
  DS_CUDA(enter_device(c->device));
  const size_t n = (size_t)dims[0] * dims[1] * dims[2];
  void *d_atoms = nullptr, *d_vals = nullptr;
  if (cudaMalloc(&d_atoms, 12ull * n_atoms) != cudaSuccess || cudaMalloc(&d_vals, 4 * n) != cudaSuccess) {
    cudaFree(d_atoms);
    return fail(DS_ERR_OOM, "build_pocket buffers");
  }
  c->allocs += 2;
  const double o[3] = {(double)origin[0], (double)origin[1], (double)origin[2]};
  const int dd[3] = {dims[0], dims[1], dims[2]};
  cudaMemcpyAsync(d_atoms, atom_xyz, 12ull * n_atoms, cudaMemcpyHostToDevice, c->stream);
  cudaEventRecord(c->ev[1], c->stream);
  launch_build_pocket((const float *)d_atoms, n_atoms, o, (double)spacing, dd, (int32_t *)d_vals, c->sm_count,
                      c->stream);
  cudaEventRecord(c->ev[2], c->stream);
  cudaMemcpyAsync(values, d_vals, 4 * n, cudaMemcpyDeviceToHost, c->stream);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess && device_ms) cudaEventElapsedTime(device_ms, c->ev[1], c->ev[2]);
  cudaFree(d_atoms);
  cudaFree(d_vals);
  if (e != cudaSuccess) return fail(DS_ERR_CUDA, "build_pocket: %s", cudaGetErrorString(e));
  return DS_OK;
}

int ds_query_capacity(ds_ctx *c, int range_idx, int *ligands) {
  if (!c || !ligands || range_idx < 0 || range_idx > 4) return fail(DS_ERR_INVALID_ARG, "bad argument");
  DS_CUDA(enter_device(c->device));
  // PAPER.md:382-384 sizes a batch as the ligands one launch keeps resident, from
  // cudaOccupancyMaxActiveBlocksPerMultiprocessor on the range's kernel.  The batched kernels here
  // give a warp to a ligand of any size (per-warp scratch for 160 atoms), so the resident ligand
  // slots are the same for every range: SMs x the smaller resident-warp count of the alignment
  // (synthetic-pocket grid in shared memory) and torsion kernels, ~90 % of the step; the select
  // kernel's residency is set by its per-warp pose slots (top-K x the batch's largest ligand),
  // which a batch does not know before it is filled.  A batch is `waves` such launches' worth
  // (DS_CAPACITY_WAVES, default 1 = the paper's one resident launch): the batched engine docks the
  // batches already waiting in one launch, so small batches cost no extra kernel tails, and the
  // first one fills (and the GPU starts) earliest with one wave.
  const int N = 8;
  const size_t per_warp = (size_t)align_warp_smem_bytes_host(N);
  const size_t grid_bytes = 181888, fixed = 30 * 16;
  int warps_a = 32;
  if (grid_bytes + fixed + per_warp * 8 <= c->smem_optin)
    warps_a = (int)std::min<size_t>(32, (c->smem_optin - grid_bytes - fixed) / per_warp);
  const int wa = warps_a * align_blocks_per_sm(warps_a, grid_bytes + fixed + per_warp * warps_a);
  const int wt = 8 * torsion_blocks_per_sm();
  cudaGetLastError();
  const int per_sm = std::min(wa, wt);
  if (per_sm <= 0) return fail(DS_ERR_CUDA, "occupancy query returned 0 resident warps");
  static const int waves = [] {
    const char *e = getenv("DS_CAPACITY_WAVES");
    const int w = e ? atoi(e) : 1;
    return w < 1 ? 1 : w;
  }();
  *ligands = c->sm_count * per_sm * waves;
  return DS_OK;
}

int ds_op_grid_score(ds_ctx *c, const ds_pocket *pk, const float *coords, int n_atoms, int n_poses, int32_t *out) {
  if (!c || !pk || !coords || !out || n_atoms < 0 || n_poses < 0) return fail(DS_ERR_INVALID_ARG, "bad argument");
  if (!n_poses) return DS_OK;
  DS_CUDA(enter_device(c->device));
  const size_t nc = 12ull * n_atoms * n_poses;
  int rc;
  if ((rc = c->ensure(c->op_in, std::max<size_t>(nc, 16))) || (rc = c->ensure(c->op_out, 4ull * n_poses))) return rc;
  DS_CUDA(cudaMemcpyAsync(c->op_in.p, coords, nc, cudaMemcpyHostToDevice, c->stream));
  launch_grid_score(pk->view, (const float *)c->op_in.p, n_atoms, n_poses, (int32_t *)c->op_out.p, c->stream);
  DS_CUDA(cudaGetLastError());
  DS_CUDA(cudaMemcpyAsync(out, c->op_out.p, 4ull * n_poses, cudaMemcpyDeviceToHost, c->stream));
  DS_CUDA(cudaStreamSynchronize(c->stream));
  return DS_OK;
}

int ds_op_rescore(ds_ctx *c, const ds_pocket *pk, const float *coords, const uint8_t *types, int n_atoms, int n_poses,
                  float cutoff, int64_t *out) {
  if (!c || !pk || !coords || !types || !out || n_atoms < 0 || n_poses < 0) return fail(DS_ERR_INVALID_ARG, "bad argument");
  if (cutoff != pk->cutoff) return fail(DS_ERR_INVALID_ARG, "cutoff must equal the last bin bound");
  if (!n_poses) return DS_OK;
  DS_CUDA(enter_device(c->device));
  const size_t nc = 12ull * n_atoms * n_poses;
  int rc;
  if ((rc = c->ensure(c->op_in, std::max<size_t>(nc, 16))) || (rc = c->ensure(c->op_aux, std::max(n_atoms, 1))) ||
      (rc = c->ensure(c->op_out, 8ull * n_poses)))
    return rc;
  DS_CUDA(cudaMemcpyAsync(c->op_in.p, coords, nc, cudaMemcpyHostToDevice, c->stream));
  DS_CUDA(cudaMemcpyAsync(c->op_aux.p, types, (size_t)n_atoms, cudaMemcpyHostToDevice, c->stream));
  launch_rescore(pk->view, (const float *)c->op_in.p, (const uint8_t *)c->op_aux.p, n_atoms, n_poses, 0.f,
                 (int64_t *)c->op_out.p, c->stream);
  DS_CUDA(cudaGetLastError());
  DS_CUDA(cudaMemcpyAsync(out, c->op_out.p, 8ull * n_poses, cudaMemcpyDeviceToHost, c->stream));
  DS_CUDA(cudaStreamSynchronize(c->stream));
  return DS_OK;
}

namespace {
// fragment arguments of the Å-frame ops: axis atoms in range and distinct, outside the mask; the
// mask within the atoms (MalformedFragment / IndexOutOfRange like validate_ligand)
int check_fragment(int n_atoms, int ab, int ae, const uint32_t *mask) {
  if (n_atoms < 1 || n_atoms > DS_MAX_ATOMS) return fail(DS_ERR_TOO_MANY_ATOMS, "n_atoms %d not in 1..%d", n_atoms, DS_MAX_ATOMS);
  if (!mask) return fail(DS_ERR_INVALID_ARG, "mask is NULL");
  if (ab < 0 || ae < 0 || ab >= n_atoms || ae >= n_atoms) return fail(DS_ERR_INDEX_OUT_OF_RANGE, "axis atom out of range");
  for (int w = 0; w < DS_MASK_WORDS; ++w) {
    const uint32_t valid = n_atoms >= 32 * (w + 1) ? 0xFFFFFFFFu : (n_atoms <= 32 * w ? 0u : ((1u << (n_atoms - 32 * w)) - 1u));
    if (mask[w] & ~valid) return fail(DS_ERR_INDEX_OUT_OF_RANGE, "mask atom out of range");
  }
  if (ab == ae || ((mask[ab >> 5] >> (ab & 31)) & 1u) || ((mask[ae >> 5] >> (ae & 31)) & 1u))
    return fail(DS_ERR_MALFORMED_FRAGMENT, "axis atoms must be distinct and outside the moving mask");
  return DS_OK;
}
}  // namespace

int ds_op_apply_rigid(ds_ctx *c, const float *coords, int n_atoms, int n_poses, const float *m, const float *center,
                      float *out) {
  if (!c || !coords || !m || !center || !out || n_atoms < 0 || n_poses < 0) return fail(DS_ERR_INVALID_ARG, "bad argument");
  if (!n_poses || !n_atoms) return DS_OK;
  DS_CUDA(enter_device(c->device));
  const size_t nc = 12ull * n_atoms * n_poses;
  int rc;
  if ((rc = c->ensure(c->op_in, nc)) || (rc = c->ensure(c->op_aux, 48ull * n_poses)) || (rc = c->ensure(c->op_out, nc)))
    return rc;
  DS_CUDA(cudaMemcpyAsync(c->op_in.p, coords, nc, cudaMemcpyHostToDevice, c->stream));
  DS_CUDA(cudaMemcpyAsync(c->op_aux.p, m, 36ull * n_poses, cudaMemcpyHostToDevice, c->stream));
  DS_CUDA(cudaMemcpyAsync((char *)c->op_aux.p + 36ull * n_poses, center, 12ull * n_poses, cudaMemcpyHostToDevice, c->stream));
  launch_apply_rigid((const float *)c->op_in.p, n_atoms, n_poses, (const float *)c->op_aux.p,
                     (const float *)((char *)c->op_aux.p + 36ull * n_poses), (float *)c->op_out.p, c->stream);
  DS_CUDA(cudaGetLastError());
  DS_CUDA(cudaMemcpyAsync(out, c->op_out.p, nc, cudaMemcpyDeviceToHost, c->stream));
  DS_CUDA(cudaStreamSynchronize(c->stream));
  return DS_OK;
}

int ds_op_apply_torsion(ds_ctx *c, const float *coords, int n_atoms, int n_poses, int axis_begin, int axis_end,
                        const uint32_t *mask, int angle_deg, float *out, int32_t *status) {
  if (!c || !coords || !out || !status || n_poses < 0) return fail(DS_ERR_INVALID_ARG, "bad argument");
  int rc;
  if ((rc = check_fragment(n_atoms, axis_begin, axis_end, mask))) return rc;
  if (!n_poses) return DS_OK;
  DS_CUDA(enter_device(c->device));
  const size_t nc = 12ull * n_atoms * n_poses;
  if ((rc = c->ensure(c->op_in, nc)) || (rc = c->ensure(c->op_out, nc)) || (rc = c->ensure(c->op_aux, 4ull * n_poses)))
    return rc;
  const int deg = ((angle_deg % 360) + 360) % 360;
  float2 cs;  // P0: the ctx's f64 -> f32 table
  DS_CUDA(cudaMemcpy(&cs, c->trig + deg, sizeof cs, cudaMemcpyDeviceToHost));
  DS_CUDA(cudaMemcpyAsync(c->op_in.p, coords, nc, cudaMemcpyHostToDevice, c->stream));
  launch_apply_torsion((const float *)c->op_in.p, n_atoms, n_poses, axis_begin, axis_end, mask, cs, deg == 0,
                       (float *)c->op_out.p, (int32_t *)c->op_aux.p, c->stream);
  DS_CUDA(cudaGetLastError());
  DS_CUDA(cudaMemcpyAsync(out, c->op_out.p, nc, cudaMemcpyDeviceToHost, c->stream));
  DS_CUDA(cudaMemcpyAsync(status, c->op_aux.p, 4ull * n_poses, cudaMemcpyDeviceToHost, c->stream));
  DS_CUDA(cudaStreamSynchronize(c->stream));
  return DS_OK;
}

int ds_op_bump_check(ds_ctx *c, const float *coords, int n_atoms, int n_poses, int axis_begin, int axis_end,
                     const uint32_t *mask, float bump_distance, int early_exit, uint8_t *bump, int64_t *pairs) {
  if (!c || !coords || !bump || !pairs || n_poses < 0 || !(bump_distance > 0.f)) return fail(DS_ERR_INVALID_ARG, "bad argument");
  int rc;
  if ((rc = check_fragment(n_atoms, axis_begin, axis_end, mask))) return rc;
  if (!n_poses) return DS_OK;
  DS_CUDA(enter_device(c->device));
  const size_t nc = 12ull * n_atoms * n_poses;
  if ((rc = c->ensure(c->op_in, nc)) || (rc = c->ensure(c->op_out, 9ull * n_poses))) return rc;
  const float bd2 = (float)((double)bump_distance * (double)bump_distance);
  DS_CUDA(cudaMemcpyAsync(c->op_in.p, coords, nc, cudaMemcpyHostToDevice, c->stream));
  long long *d_pairs = (long long *)c->op_out.p;
  uint8_t *d_bump = (uint8_t *)(d_pairs + n_poses);
  launch_bump_check((const float *)c->op_in.p, n_atoms, n_poses, axis_begin, axis_end, mask, bd2, early_exit ? 1 : 0,
                    d_bump, d_pairs, c->stream);
  DS_CUDA(cudaGetLastError());
  DS_CUDA(cudaMemcpyAsync(pairs, d_pairs, 8ull * n_poses, cudaMemcpyDeviceToHost, c->stream));
  DS_CUDA(cudaMemcpyAsync(bump, d_bump, (size_t)n_poses, cudaMemcpyDeviceToHost, c->stream));
  DS_CUDA(cudaStreamSynchronize(c->stream));
  return DS_OK;
}

}  // extern "C"
