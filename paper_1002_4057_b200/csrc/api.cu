// C-ABI of the B200 SPD tile-inversion engine (include/tileinv_b200.h):
// device tile store, layout conversion, native stream generation
// (taskgen.py), the hazard scoreboard (scheduler.py:101-153), the planner
// that turns a stream into a device-resident DAG, and the executor launch.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <map>
#include <queue>
#include <unordered_map>
#include <vector>

#include "tinv_internal.h"
#include "host_plan.h"

namespace tinv {
cudaError_t launch_exec(const CUtensorMap& tmK, const CUtensorMap& tmM, const CUtensorMap& tmE, const ExecParams& P,
                        int b, int grid, cudaStream_t stream);
cudaError_t launch_put(const double* src, int64_t lda, int64_t row0, double* pool, int64_t slot_elems,
                       const int32_t* slot_of, int b, int bp, int64_t tri_lo, int64_t ntiles, cudaStream_t st,
                       int64_t T1, int64_t mstride);
cudaError_t launch_get(double* dst, int64_t ldd, int64_t row0, const double* pool, int64_t slot_elems,
                       const int32_t* slot_of, int b, int bp, int t, int panel_i, int64_t tile_lo,
                       int64_t ntiles, int symmetrize, cudaStream_t st, int64_t T1, int64_t mstride);
cudaError_t launch_copy_slots(double* pool, int64_t slot_elems, const int32_t* from, const int32_t* to,
                              int64_t n, cudaStream_t st);
cudaError_t launch_pad(double* pool, int64_t slot_elems, const int32_t* slot_of, int b, int bp, int64_t ntiles,
                       int64_t T1, cudaStream_t st);
}  // namespace tinv

using namespace tinv;

static std::string g_err;
// executor tunables (environment overrides for experiments):
// fetch-and-add claims on ready levels with at least this backlog (TINV_TICKET_MIN)
static const int kTicketMin = 64;
// next-item claim ahead of time from levels with at least this backlog; 0 = off
// (TINV_PREFETCH_MIN; measured: hurts C2's critical path, neutral on C3)
static const int kPrefetchMin = 0;
// bottom-level weight of a streamed-output departure in b^3 units (TINV_DEPART_WEIGHT)
static const double kDepartWeight = 0.0;


#define CK(ctx, call)                                                                               \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess) {                                                                        \
      std::string m_ = std::string(#call) + ": " + cudaGetErrorString(e_);                          \
      if (ctx) (ctx)->err = m_;                                                                     \
      g_err = m_;                                                                                   \
      return TINV_ERR_CUDA;                                                                         \
    }                                                                                               \
  } while (0)

namespace tinv {
int set_error(int code, const std::string& msg) {  // error text for context-free entry points (batched.cu)
  g_err = msg;
  return code;
}
}  // namespace tinv

static int fail(tinv_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  g_err = msg;
  return code;
}

// ------------------------------------------------------------------ tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// the other slot of lower tile k's pair (home slot, shadow: T + k, or compact in a partitioned store)
static inline int32_t alt_slot_of(const tinv_ctx* c, int64_t k) {
  return c->a_slot[k] == c->home[k] ? c->shadow[k] : c->home[k];
}

static int make_maps(tinv_ctx* c) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    CK(c, cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) return fail(c, TINV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)p;
  }
  cuuint64_t dims[3] = {(cuuint64_t)c->bp, (cuuint64_t)c->bp, (cuuint64_t)c->pool_slots};
  cuuint64_t strides[2] = {(cuuint64_t)c->bp * 8, (cuuint64_t)c->bp * c->bp * 8};
  cuuint32_t estr[3] = {1, 1, 1};
  cuuint32_t boxK[3] = {KCH, BLK, 1};  // 16 doubles (128 B) x 128 rows
  cuuint32_t boxM[3] = {16, KCH, 1};   // 16 doubles x 16 rows
  cuuint32_t boxE[3] = {16, 32, 1};    // epilogue: 16 doubles x 32 rows
  CUresult r1 = fn(&c->tmK, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->pool, dims, strides, boxK, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = fn(&c->tmM, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->pool, dims, strides, boxM, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r3 = fn(&c->tmE, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->pool, dims, strides, boxE, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS || r3 != CUDA_SUCCESS)
    return fail(c, TINV_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r1) + "/" + std::to_string(r2));
  return TINV_OK;
}

// grow the slot pool to at least `slots`, keeping the matrix region [0, 2T)
static int ensure_pool(tinv_ctx* c, int64_t slots) {
  if (slots <= c->pool_slots) return TINV_OK;
  if (c->exported) return fail(c, TINV_ERR_BAD_ARG, "tile store is mapped by peer ranks and cannot grow");
  CK(c, cudaSetDevice(c->device));
  double* np = nullptr;
  CK(c, cudaMalloc(&np, (size_t)slots * c->slot_elems * 8));
  if (c->pool) {
    CK(c, cudaMemcpyAsync(np, c->pool, (size_t)std::min<int64_t>(c->pool_slots, c->mslots) * c->slot_elems * 8,
                          cudaMemcpyDeviceToDevice, c->st));
    CK(c, cudaStreamSynchronize(c->st));
    CK(c, cudaFree(c->pool));
  }
  c->pool = np;
  c->pool_slots = slots;
  return make_maps(c);
}

// ------------------------------------------------------------------ C-ABI: context
extern "C" {

int tinv_abi_version(void) { return TINV_ABI_VERSION; }

const char* tinv_last_error(const tinv_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

int tinv_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int ok = 0;
  for (int d = 0; d < n; ++d) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++ok;
  }
  return ok;
}

int tinv_create(tinv_ctx** out, int64_t n, int64_t b, int device) { return tinv_create_batch(out, 1, n, b, device); }

static int create_impl(tinv_ctx** out, int64_t batch, int64_t n, int64_t b, int device, const int32_t* owned);

int tinv_create_batch(tinv_ctx** out, int64_t batch, int64_t n, int64_t b, int device) {
  return create_impl(out, batch, n, b, device, nullptr);
}

int tinv_create_owned(tinv_ctx** out, int64_t n, int64_t b, int device, const int32_t* owned) {
  if (!owned) return fail(nullptr, TINV_ERR_BAD_ARG, "null ownership mask");
  return create_impl(out, 1, n, b, device, owned);
}

static int create_impl(tinv_ctx** out, int64_t batch, int64_t n, int64_t b, int device, const int32_t* owned) {
  if (!out) return fail(nullptr, TINV_ERR_BAD_ARG, "null ctx pointer");
  *out = nullptr;
  if (n < 1 || b < 1 || n % b) return fail(nullptr, TINV_ERR_BAD_ARG, "matrix order not divisible by tile order");
  if (batch < 1) return fail(nullptr, TINV_ERR_BAD_ARG, "batch must be >= 1");
  int nd = 0;
  if (cudaGetDeviceCount(&nd) != cudaSuccess || device < 0 || device >= nd) {
    cudaGetLastError();
    return fail(nullptr, TINV_ERR_NO_DEVICE, "no CUDA device");
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10)
    return fail(nullptr, TINV_ERR_NO_DEVICE, "device is not sm_100 (B200)");
  tinv_ctx* c = new tinv_ctx();
  c->n = n;
  c->b = b;
  c->t = n / b;
  c->bp = (b + BLK - 1) / BLK * BLK;
  c->R = c->bp / BLK;
  c->T1 = c->t * (c->t + 1) / 2;
  c->nmat = batch;
  c->T = c->T1 * batch;
  c->device = device;
  c->nsm = prop.multiProcessorCount;
  c->slot_elems = c->bp * c->bp;
  int rc = TINV_OK;
  auto bail = [&](int code) {
    tinv_destroy(c);
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) return bail(fail(nullptr, TINV_ERR_CUDA, "cudaSetDevice failed"));
  if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(nullptr, TINV_ERR_CUDA, "stream create failed"));
  c->own = c->st;
  c->a_slot.resize(c->T);
  c->home.resize(c->T);
  c->shadow.resize(c->T);
  if (!owned) {
    for (int64_t k = 0; k < c->T; ++k) c->a_slot[k] = c->home[k] = (int32_t)k, c->shadow[k] = (int32_t)(c->T + k);
    c->mslots = 2 * c->T;
  } else {  // partitioned: slots only for this rank's tiles (owned[i * t + j], i >= j), homes then shadows
    c->partitioned = true;
    int64_t nown = 0;
    for (int64_t i = 0; i < c->t; ++i)
      for (int64_t j = 0; j <= i; ++j) nown += owned[i * c->t + j] != 0;
    int32_t s = 0;
    for (int64_t i = 0; i < c->t; ++i)
      for (int64_t j = 0; j <= i; ++j) {
        const int64_t k = tri_index(i, j);
        const bool mine = owned[i * c->t + j] != 0;
        c->a_slot[k] = c->home[k] = mine ? s : -1;
        c->shadow[k] = mine ? (int32_t)(nown + s) : -1;
        s += mine;
      }
    c->mslots = 2 * nown;
  }
  if (cudaMalloc(&c->d_a_slot, c->T * sizeof(int32_t)) != cudaSuccess)
    return bail(fail(nullptr, TINV_ERR_CUDA, "cudaMalloc failed"));
  cudaMemcpy(c->d_a_slot, c->a_slot.data(), c->T * sizeof(int32_t), cudaMemcpyHostToDevice);
  rc = ensure_pool(c, c->mslots + c->nsm);
  if (rc != TINV_OK) {
    g_err = c->err;
    return bail(rc);
  }
  *out = c;
  return TINV_OK;
}

int tinv_destroy(tinv_ctx* c) {
  if (!c) return TINV_OK;
  cudaSetDevice(c->device);
  if (c->pool) cudaFree(c->pool);
  if (c->d_a_slot) cudaFree(c->d_a_slot);
  if (c->bstage) cudaFree(c->bstage);
  for (int r = 0; r < MAX_RANKS && !c->attached; ++r) {
    if (r == c->rank) continue;
    if (c->peer_pool[r]) cudaIpcCloseMemHandle(c->peer_pool[r]);
    if (c->peer_inbox[r]) cudaIpcCloseMemHandle(c->peer_inbox[r]);
  }
  if (c->inbox) cudaFree(c->inbox);
  for (auto& s : c->staging)
    if (s) cudaFree(s);
  if (c->own) cudaStreamDestroy(c->own);
  if (c->st2) cudaStreamDestroy(c->st2);
  for (cudaStream_t s : c->dst)
    if (s) cudaStreamDestroy(s);
  delete c;
  return TINV_OK;
}

int tinv_set_stream(tinv_ctx* c, void* stream) {
  if (!c) return TINV_ERR_BAD_ARG;
  c->st = stream ? (cudaStream_t)stream : c->own;
  return TINV_OK;
}

int tinv_store_bytes(const tinv_ctx* c, int64_t* bytes) {
  if (!c || !bytes) return TINV_ERR_BAD_ARG;
  *bytes = c->pool_slots * c->slot_elems * 8;
  return TINV_OK;
}

int tinv_shape(const tinv_ctx* c, int64_t* n, int64_t* b, int64_t* t, int64_t* bp) {
  if (!c) return TINV_ERR_BAD_ARG;
  if (n) *n = c->n;
  if (b) *b = c->b;
  if (t) *t = c->t;
  if (bp) *bp = c->bp;
  return TINV_OK;
}

static int ensure_staging(tinv_ctx* c) {
  const size_t need = (size_t)c->b * c->n * 8;
  if (c->staging_bytes >= need) return TINV_OK;
  for (auto& s : c->staging) {
    if (s) cudaFree(s);
    s = nullptr;
    CK(c, cudaMalloc(&s, need));
  }
  c->staging_bytes = need;
  return TINV_OK;
}

static int sync_slots(tinv_ctx* c) {
  CK(c, cudaMemcpyAsync(c->d_a_slot, c->a_slot.data(), c->T * sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
  return TINV_OK;
}

int tinv_put_dense_device(tinv_ctx* c, const double* dev, int64_t lda) {
  if (!c || !dev || lda < c->n) return fail(c, TINV_ERR_BAD_ARG, "bad put_dense_device arguments");
  CK(c, cudaSetDevice(c->device));
  int rc = sync_slots(c);
  if (rc) return rc;
  CK(c, launch_put(dev, lda, 0, c->pool, c->slot_elems, c->d_a_slot, (int)c->b, (int)c->bp, 0, c->T, c->st, c->T1,
                   c->n * lda));
  CK(c, cudaStreamSynchronize(c->st));
  return TINV_OK;
}

int tinv_get_dense_device(tinv_ctx* c, double* dev, int64_t lda, int mode) {
  if (!c || !dev || lda < c->n) return fail(c, TINV_ERR_BAD_ARG, "bad get_dense_device arguments");
  CK(c, cudaSetDevice(c->device));
  int rc = sync_slots(c);
  if (rc) return rc;
  const int sym = mode == TINV_DENSE_SYMMETRIZE;
  // SYMMETRIZE on the device: each lower tile read once, written with its mirror (mode 2)
  CK(c, launch_get(dev, lda, 0, c->pool, c->slot_elems, c->d_a_slot, (int)c->b, (int)c->bp, (int)c->t, -1, 0,
                   c->T, sym ? 2 : 0, c->st, c->T1, c->n * lda));
  CK(c, cudaStreamSynchronize(c->st));
  return TINV_OK;
}

// Host transfers go by tile-row panels through two device staging buffers:
// H2D of panel i+1 (copy stream) overlaps the conversion of panel i.
static int ensure_bstage(tinv_ctx* c) {
  if (c->bstage) return TINV_OK;
  CK(c, cudaMalloc(&c->bstage, (size_t)c->nmat * c->n * c->n * 8));
  return TINV_OK;
}

// partitioned store (tinv_create_owned): only this rank's tiles cross PCIe,
// one 2D copy per owned tile straight into its slot (+ the closure padding)
static int put_owned_tiles(tinv_ctx* c, const double* host, int64_t lda) {
  int rc = sync_slots(c);
  if (rc) return rc;
  const int64_t b = c->b, bp = c->bp;
  for (int64_t i = 0; i < c->t; ++i)
    for (int64_t j = 0; j <= i; ++j) {
      const int32_t sl = c->a_slot[tri_index(i, j)];
      if (sl < 0) continue;
      CK(c, cudaMemcpy2DAsync(c->pool + (int64_t)sl * c->slot_elems, bp * 8, host + i * b * lda + j * b, lda * 8,
                              b * 8, b, cudaMemcpyHostToDevice, c->st));
    }
  if (bp != b) CK(c, launch_pad(c->pool, c->slot_elems, c->d_a_slot, (int)b, (int)bp, c->T, c->T1, c->st));
  CK(c, cudaStreamSynchronize(c->st));
  return TINV_OK;
}

static int get_owned_tiles(tinv_ctx* c, double* host, int64_t lda, int mode) {
  if (mode != TINV_DENSE_LOWER_TILES) return fail(c, TINV_ERR_BAD_ARG, "a partitioned store returns its own lower tiles only");
  int rc = sync_slots(c);
  if (rc) return rc;
  const int64_t b = c->b, bp = c->bp;
  for (int64_t i = 0; i < c->t; ++i)
    for (int64_t j = 0; j <= i; ++j) {
      const int32_t sl = c->a_slot[tri_index(i, j)];
      if (sl < 0) continue;
      CK(c, cudaMemcpy2DAsync(host + i * b * lda + j * b, lda * 8, c->pool + (int64_t)sl * c->slot_elems, bp * 8,
                              b * 8, b, cudaMemcpyDeviceToHost, c->st));
    }
  CK(c, cudaStreamSynchronize(c->st));
  return TINV_OK;
}

int tinv_put_dense(tinv_ctx* c, const double* host, int64_t lda) {
  if (!c || !host || lda < c->n) return fail(c, TINV_ERR_BAD_ARG, "bad put_dense arguments");
  CK(c, cudaSetDevice(c->device));
  if (c->partitioned) return put_owned_tiles(c, host, lda);
  if (c->nmat > 1) {  // batch: one bulk copy of all matrices, then one conversion
    int rc = ensure_bstage(c);
    if (rc) return rc;
    CK(c, cudaMemcpy2DAsync(c->bstage, c->n * 8, host, lda * 8, c->n * 8, c->nmat * c->n, cudaMemcpyHostToDevice,
                            c->st));
    return tinv_put_dense_device(c, c->bstage, c->n);
  }
  int rc = ensure_staging(c);
  if (rc) return rc;
  rc = sync_slots(c);
  if (rc) return rc;
  cudaEvent_t copied[2], freed[2];
  for (int k = 0; k < 2; ++k) {
    CK(c, cudaEventCreateWithFlags(&copied[k], cudaEventDisableTiming));
    CK(c, cudaEventCreateWithFlags(&freed[k], cudaEventDisableTiming));
    CK(c, cudaEventRecord(freed[k], c->st));
  }
  const int64_t b = c->b, n = c->n;
  for (int64_t i = 0; i < c->t; ++i) {
    const int k = (int)(i & 1);
    CK(c, cudaStreamWaitEvent(c->st2, freed[k], 0));
    CK(c, cudaMemcpy2DAsync(c->staging[k], n * 8, host + i * b * lda, lda * 8, (size_t)(i + 1) * b * 8, b,
                            cudaMemcpyHostToDevice, c->st2));
    CK(c, cudaEventRecord(copied[k], c->st2));
    CK(c, cudaStreamWaitEvent(c->st, copied[k], 0));
    CK(c, launch_put(c->staging[k], n, i * b, c->pool, c->slot_elems, c->d_a_slot, (int)b, (int)c->bp,
                     tri_index(i, 0), i + 1, c->st, c->T1, 0));
    CK(c, cudaEventRecord(freed[k], c->st));
  }
  CK(c, cudaStreamSynchronize(c->st));
  CK(c, cudaStreamSynchronize(c->st2));
  for (int k = 0; k < 2; ++k) {
    cudaEventDestroy(copied[k]);
    cudaEventDestroy(freed[k]);
  }
  return TINV_OK;
}

int tinv_get_dense(tinv_ctx* c, double* host, int64_t lda, int mode) {
  if (!c || !host || lda < c->n) return fail(c, TINV_ERR_BAD_ARG, "bad get_dense arguments");
  CK(c, cudaSetDevice(c->device));
  if (c->partitioned) return get_owned_tiles(c, host, lda, mode);
  if (c->nmat > 1) {
    int rc = ensure_bstage(c);
    if (rc) return rc;
    if (mode != TINV_DENSE_SYMMETRIZE)  // LOWER mode keeps the caller's upper tiles
      CK(c, cudaMemcpy2DAsync(c->bstage, c->n * 8, host, lda * 8, c->n * 8, c->nmat * c->n, cudaMemcpyHostToDevice,
                              c->st));
    rc = tinv_get_dense_device(c, c->bstage, c->n, mode);
    if (rc) return rc;
    CK(c, cudaMemcpy2DAsync(host, lda * 8, c->bstage, c->n * 8, c->n * 8, c->nmat * c->n, cudaMemcpyDeviceToHost,
                            c->st));
    CK(c, cudaStreamSynchronize(c->st));
    return TINV_OK;
  }
  int rc = ensure_staging(c);
  if (rc) return rc;
  rc = sync_slots(c);
  if (rc) return rc;
  const int sym = mode == TINV_DENSE_SYMMETRIZE;
  cudaEvent_t built[2], freed[2];
  for (int k = 0; k < 2; ++k) {
    CK(c, cudaEventCreateWithFlags(&built[k], cudaEventDisableTiming));
    CK(c, cudaEventCreateWithFlags(&freed[k], cudaEventDisableTiming));
    CK(c, cudaEventRecord(freed[k], c->st2));
  }
  const int64_t b = c->b, n = c->n;
  for (int64_t i = 0; i < c->t; ++i) {
    const int k = (int)(i & 1);
    const int64_t ntile = sym ? c->t : i + 1;
    CK(c, cudaStreamWaitEvent(c->st, freed[k], 0));
    CK(c, launch_get(c->staging[k], n, i * b, c->pool, c->slot_elems, c->d_a_slot, (int)b, (int)c->bp,
                     (int)c->t, (int)i, 0, ntile, sym, c->st, c->T1, 0));
    CK(c, cudaEventRecord(built[k], c->st));
    CK(c, cudaStreamWaitEvent(c->st2, built[k], 0));
    CK(c, cudaMemcpy2DAsync(host + i * b * lda, lda * 8, c->staging[k], n * 8, (size_t)ntile * b * 8, b,
                            cudaMemcpyDeviceToHost, c->st2));
    CK(c, cudaEventRecord(freed[k], c->st2));
  }
  CK(c, cudaStreamSynchronize(c->st));
  CK(c, cudaStreamSynchronize(c->st2));
  for (int k = 0; k < 2; ++k) {
    cudaEventDestroy(built[k]);
    cudaEventDestroy(freed[k]);
  }
  return TINV_OK;
}

int tinv_put_tile(tinv_ctx* c, int64_t i, int64_t j, const double* host) {
  if (!c || !host || i < 0 || j < 0 || j > i || i >= c->t) return fail(c, TINV_ERR_BAD_ARG, "bad tile index");
  CK(c, cudaSetDevice(c->device));
  int rc = sync_slots(c);
  if (rc) return rc;
  const int64_t b = c->b, bp = c->bp, x = tri_index(i, j);
  if (c->a_slot[x] < 0) return fail(c, TINV_ERR_BAD_ARG, "tile of another rank's store");
  double* slot = c->pool + (int64_t)c->a_slot[x] * c->slot_elems;
  // the b x b tile straight into its slot; a padded slot (bp > b) gets the
  // closure padding (identity on a diagonal tile, 0 elsewhere) around it
  if (bp != b) {
    if (i == j)  // one-tile pad launch: slot_of = this tile's slot entry, decoded as a diagonal tile
      CK(c, launch_pad(c->pool, c->slot_elems, c->d_a_slot + x, (int)b, (int)bp, 1, 1, c->st));
    else
      CK(c, cudaMemset2DAsync(slot, bp * 8, 0, bp * 8, bp, c->st));
  }
  CK(c, cudaMemcpy2DAsync(slot, bp * 8, host, b * 8, b * 8, b, cudaMemcpyHostToDevice, c->st));
  CK(c, cudaStreamSynchronize(c->st));
  return TINV_OK;
}

int tinv_get_tile(tinv_ctx* c, int64_t i, int64_t j, double* host) {
  if (!c || !host || i < 0 || j < 0 || j > i || i >= c->t) return fail(c, TINV_ERR_BAD_ARG, "bad tile index");
  CK(c, cudaSetDevice(c->device));
  const int64_t b = c->b;
  if (c->a_slot[tri_index(i, j)] < 0) return fail(c, TINV_ERR_BAD_ARG, "tile of another rank's store");
  CK(c, cudaMemcpy2D(host, b * 8, c->pool + (int64_t)c->a_slot[tri_index(i, j)] * c->slot_elems, c->bp * 8, b * 8,
                     b, cudaMemcpyDeviceToHost));
  return TINV_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ streams and DAGs
namespace {

struct Tk {
  int32_t f[TINV_TASK_FIELDS];
};

enum { F_KIND, F_STEP, F_I, F_J, F_K, F_OL, F_OR, F_OC, F_OM, F_NR, F_R0L, F_R0R, F_R0C, F_R1L, F_R1R, F_R1C };

struct Gen {
  std::vector<Tk> tasks;
  void add(int kind, int step, int i, int j, int k, int ol, int orr, int oc, int mode, int nr, int r0l = -1,
           int r0r = -1, int r0c = -1, int r1l = -1, int r1r = -1, int r1c = -1) {
    Tk t = {{kind, step, i, j, k, ol, orr, oc, mode, nr, r0l, r0r, r0c, r1l, r1r, r1c}};
    tasks.push_back(t);
  }
  // taskgen.py:164-170
  void copies(int t, int src, int dst) {
    for (int r = 0; r < t; ++r)
      for (int c = 0; c <= r; ++c) add(TINV_COPY, TINV_STEP_COPY, r, c, -1, dst, r, c, 2, 1, src, r, c);
  }
  // taskgen.py:178-189
  void step1(int t, char d) {
    for (int j = 0; j < t; ++j) {
      for (int k = 0; k < j; ++k) add(TINV_SYRK_SUB, 1, j, k, -1, 0, j, j, 1, 1, 0, j, k);
      add(TINV_POTRF, 1, j, -1, -1, 0, j, j, 1, 0);
      for (int i = j + 1; i < t; ++i)
        for (int s = 0; s < j; ++s) {
          const int k = d == 'U' ? s : j - 1 - s;
          add(TINV_GEMM, 1, i, j, k, 0, i, j, 1, 2, 0, i, k, 0, j, k);
        }
      for (int i = j + 1; i < t; ++i) add(TINV_TRSM, 1, i, j, -1, 0, i, j, 1, 1, 0, j, j);
    }
  }
  // taskgen.py:192-205
  void step2(int t, char d, bool oop) {
    if (oop && t > 1) copies(t, 0, 1);
    const int col = oop ? 1 : 0;
    for (int j = t - 1; j >= 0; --j) {
      add(TINV_TRTRI, 2, j, -1, -1, 0, j, j, 1, 0);
      for (int i = t - 1; i > j; --i) {
        add(TINV_TRMM_LEFT, 2, i, j, -1, 0, i, j, 1, 1, 0, i, i);
        const int lo = j + 1, hi = i;
        for (int s = 0; s < hi - lo; ++s) {
          const int k = d == 'U' ? lo + s : hi - 1 - s;
          add(TINV_GEMM, 2, i, j, k, 0, i, j, 1, 2, 0, i, k, col, k, j);
        }
        add(TINV_TRMM_RIGHT_NEG, 2, i, j, -1, 0, i, j, 1, 1, 0, j, j);
      }
    }
  }
  // taskgen.py:208-223
  void step3(int t, char d, bool oop) {
    if (oop && t > 1) copies(t, 0, 2);
    const int src = oop ? 2 : 0;
    for (int i = 0; i < t; ++i) {
      for (int j = 0; j < i; ++j) add(TINV_TRMM_LEFT_T, 3, i, j, -1, 0, i, j, 1, 1, src, i, i);
      add(TINV_LAUUM, 3, i, -1, -1, 0, i, i, 1, 0);
      for (int j = 0; j < i; ++j) {
        const int lo = i + 1, hi = t;
        for (int s = 0; s < hi - lo; ++s) {
          const int k = d == 'U' ? lo + s : hi - 1 - s;
          add(TINV_GEMM, 3, i, j, k, 0, i, j, 1, 2, src, k, i, src, k, j);
        }
      }
      for (int k = i + 1; k < t; ++k) add(TINV_SYRK_ADD_T, 3, i, k, -1, 0, i, i, 1, 1, src, k, i);
    }
  }
};

// accesses of a task: reads (operand order) then the output
struct Acc {
  int64_t tile;
  int mode;  // 0 R, 1 RW, 2 W
};

struct Edge {
  int32_t u, v;
  int8_t kind;  // 0 RAW 1 WAR 2 WAW 3 barrier
};

// Scoreboard of scheduler.py:101-140 over abstract tile keys + barrier edges
// (scheduler.py:143-153: prefix sinks -> suffix sources).
void scoreboard(int64_t n, const std::vector<std::vector<Acc>>& acc, const std::vector<int64_t>& barriers,
                std::vector<Edge>& edges) {
  std::unordered_map<int64_t, int32_t> last_writer;
  std::unordered_map<int64_t, std::vector<int32_t>> readers;
  last_writer.reserve(n * 2);
  readers.reserve(n * 2);
  std::vector<std::pair<int32_t, int64_t>> raw;
  for (int64_t v = 0; v < n; ++v) {
    raw.clear();
    for (const Acc& a : acc[v])
      if (a.mode == 0 || a.mode == 1) {
        auto it = last_writer.find(a.tile);
        if (it != last_writer.end()) {
          edges.push_back({it->second, (int32_t)v, 0});
          raw.push_back({it->second, a.tile});
        }
      }
    for (const Acc& a : acc[v])
      if (a.mode == 1 || a.mode == 2) {
        auto rit = readers.find(a.tile);
        if (rit != readers.end())
          for (int32_t r : rit->second) edges.push_back({r, (int32_t)v, 1});
        auto it = last_writer.find(a.tile);
        if (it != last_writer.end()) {
          bool has = false;
          for (auto& p : raw)
            if (p.first == it->second && p.second == a.tile) has = true;
          if (!has) edges.push_back({it->second, (int32_t)v, 2});
        }
      }
    for (const Acc& a : acc[v])
      if (a.mode == 0 || a.mode == 1) readers[a.tile].push_back((int32_t)v);
    for (const Acc& a : acc[v])
      if (a.mode == 1 || a.mode == 2) {
        last_writer[a.tile] = (int32_t)v;
        readers[a.tile].clear();
      }
  }
  std::vector<int64_t> bs(barriers);
  std::sort(bs.begin(), bs.end());
  for (int64_t pos : bs) {
    std::vector<char> has_out(n, 0), has_in(n, 0);
    for (const Edge& e : edges) {
      if (e.u < pos && e.v < pos) has_out[e.u] = 1;
      if (e.u >= pos && e.v >= pos) has_in[e.v] = 1;
    }
    std::vector<int32_t> sinks, sources;
    for (int64_t u = 0; u < std::min<int64_t>(pos, n); ++u)
      if (!has_out[u]) sinks.push_back((int32_t)u);
    for (int64_t v = std::max<int64_t>(pos, 0); v < n; ++v)
      if (!has_in[v]) sources.push_back((int32_t)v);
    for (int32_t u : sinks)
      for (int32_t v : sources) edges.push_back({u, v, 3});
  }
}

int64_t tile_key(int label, int r, int c) { return ((int64_t)label << 36) | ((int64_t)r << 18) | (int64_t)c; }

void ref_accesses(const int32_t* table, int64_t n, std::vector<std::vector<Acc>>& acc) {
  acc.resize(n);
  for (int64_t v = 0; v < n; ++v) {
    const int32_t* f = table + v * TINV_TASK_FIELDS;
    acc[v].clear();
    if (f[F_NR] >= 1) acc[v].push_back({tile_key(f[F_R0L], f[F_R0R], f[F_R0C]), 0});
    if (f[F_NR] >= 2) acc[v].push_back({tile_key(f[F_R1L], f[F_R1R], f[F_R1C]), 0});
    acc[v].push_back({tile_key(f[F_OL], f[F_OR], f[F_OC]), f[F_OM] == 2 ? 2 : 1});
  }
}

int expected_reads(int kind) {
  switch (kind) {
    case TINV_POTRF:
    case TINV_TRTRI:
    case TINV_LAUUM:
    case KIND_RECV:
      return 0;
    case TINV_GEMM:
      return 2;
    default:
      return 1;
  }
}

double weight_of(int kind) {  // flops in units of b^3 (SURVEY.md §7 hard part 2)
  switch (kind) {
    case KIND_POTRF_INV:
      return 2.0 / 3.0;  // factor + the factor's inverse
    case TINV_POTRF:
    case TINV_TRTRI:
    case TINV_LAUUM:
    case KIND_INV:
      return 1.0 / 3.0;
    case TINV_GEMM:
      return 2.0;
    case TINV_COPY:
      return 0.05;
    case KIND_ARRIVE:
    case KIND_DEPART:
      return 0.0;
    default:
      return 1.0;
  }
}

// Critical-path length estimate of a task in units of one 128^3 block product
// on one SM (~17 us): item phases run one after another, the items of a phase
// in parallel. The diagonal chains dominate when the DAG is latency-bound
// (C2: a POTRF of a 256 tile takes ~5x a GEMM of the same tile although it
// does a sixth of its flops), so bottom levels in flops under-prioritise them.
// latency of a mirrored (symmetric-output) block item beyond its block
// products, in block-product units (TINV_MIRROR_COST). Measured at C2: a
// mirrored SYRK_ADD_T item takes 69 us against 46 us for a GEMM item of the
// same K; weighting it 2.5 (GEMM: 0.5) puts step 3's diagonal accumulation
// chains -- the DAG's tail -- ahead of the off-diagonal ones: 19.14 -> 18.94 ms
// (0.5 / 1.0 / 1.5 / 2.5: 19.14 / 19.05 / 19.08 / 18.94 ms).
static double mirror_cost() {
  static const double v = getenv("TINV_MIRROR_COST") ? atof(getenv("TINV_MIRROR_COST")) : 2.5;
  return v;
}

double latency_of(int kind, int R, int flags = 0) {
  const double r = R;
  switch (kind) {
    case KIND_POTRF_INV:  // R factor+inverse blocks, TRSM / update phases, the full inverse
      return 4.0 * r + (r - 1.0) * r + r;
    case TINV_POTRF:
      return 4.0 * r + (r - 1.0) * r;
    case TINV_TRTRI:
    case KIND_INV:
      return 1.5 * r + (r - 1.0) * r;
    case TINV_COPY:
      return 0.3;
    case KIND_ARRIVE:
    case KIND_DEPART:
      return 0.0;
    case TINV_SYRK_ADD_T:  // symmetric outputs: the generic epilogue with the mirror (C2: 69 us an item
    case TINV_LAUUM:       // against 46 us for a GEMM of the same K)
      return r + mirror_cost();
    case TINV_SYRK_SUB:
      return r + ((flags & TF_NO_MIRROR) ? 0.5 : mirror_cost());
    default:  // GEMM, TRSM, TRMM: one phase of K <= R block products
      return r + 0.5;
  }
}

}  // namespace

// ------------------------------------------------------------------ plans

extern "C" {

int tinv_gen_stream(int32_t t, int32_t steps, const char* loops, int32_t out_of_place, int32_t pipelined,
                    int32_t* table, int64_t cap, int64_t* ntasks, int64_t* barriers, int64_t capb, int64_t* nbar) {
  if (t < 1 || steps < 1 || steps > 7 || !loops) return fail(nullptr, TINV_ERR_BAD_ARG, "bad gen_stream arguments");
  const size_t nl = strlen(loops);
  for (size_t x = 0; x < nl; ++x)
    if (loops[x] != 'U' && loops[x] != 'D') return fail(nullptr, TINV_ERR_BAD_ARG, "loop order must be [UD]");
  Gen g;
  std::vector<int64_t> bars;
  int nsteps = 0;
  for (int s = 0; s < 3; ++s) nsteps += (steps >> s) & 1;
  int which = 0;
  for (int s = 0; s < 3; ++s) {
    if (!((steps >> s) & 1)) continue;
    const char d = nsteps > 1 ? loops[std::min<size_t>(s, nl - 1)] : loops[0];
    if (which > 0 && !pipelined) bars.push_back((int64_t)g.tasks.size());
    if (s == 0) g.step1(t, d);
    if (s == 1) g.step2(t, d, out_of_place != 0);
    if (s == 2) g.step3(t, d, out_of_place != 0);
    ++which;
  }
  if (ntasks) *ntasks = (int64_t)g.tasks.size();
  if (nbar) *nbar = (int64_t)bars.size();
  if (table) {
    if (cap < (int64_t)g.tasks.size()) return fail(nullptr, TINV_ERR_BAD_ARG, "table capacity too small");
    memcpy(table, g.tasks.data(), g.tasks.size() * sizeof(Tk));
  }
  if (barriers) {
    if (capb < (int64_t)bars.size()) return fail(nullptr, TINV_ERR_BAD_ARG, "barrier capacity too small");
    for (size_t x = 0; x < bars.size(); ++x) barriers[x] = bars[x];
  }
  return TINV_OK;
}

int tinv_dag_edges(const int32_t* table, int64_t n, const int64_t* barriers, int64_t nbar, int32_t* src,
                   int32_t* dst, int8_t* kind, int64_t cap, int64_t* nedges) {
  if (!table && n > 0) return fail(nullptr, TINV_ERR_BAD_ARG, "null table");
  std::vector<std::vector<Acc>> acc;
  ref_accesses(table, n, acc);
  std::vector<int64_t> bars(barriers, barriers + (barriers ? nbar : 0));
  std::vector<Edge> edges;
  scoreboard(n, acc, bars, edges);
  if (nedges) *nedges = (int64_t)edges.size();
  if (src) {
    if (cap < (int64_t)edges.size()) return fail(nullptr, TINV_ERR_BAD_ARG, "edge capacity too small");
    for (size_t x = 0; x < edges.size(); ++x) {
      src[x] = edges[x].u;
      dst[x] = edges[x].v;
      kind[x] = edges[x].kind;
    }
  }
  return TINV_OK;
}

int tinv_dag_paths(const int32_t* table, int64_t n, const int64_t* barriers, int64_t nbar, const double* weight,
                   int32_t include_copies, double* best, int32_t* via, int32_t* depth, int64_t* ncomp) {
  if ((!table && n > 0) || n < 0) return fail(nullptr, TINV_ERR_BAD_ARG, "null table");
  std::vector<std::vector<Acc>> acc;
  ref_accesses(table, n, acc);
  std::vector<int64_t> bars(barriers, barriers + (barriers ? nbar : 0));
  std::vector<Edge> edges;
  scoreboard(n, acc, bars, edges);
  // predecessor lists in ascending id (dedup): CSR by destination
  std::vector<int64_t> off(n + 1, 0);
  for (const Edge& e : edges) off[e.v + 1]++;
  for (int64_t v = 0; v < n; ++v) off[v + 1] += off[v];
  std::vector<int32_t> pred(edges.size());
  {
    std::vector<int64_t> fill(off.begin(), off.end() - 1);
    for (const Edge& e : edges) pred[fill[e.v]++] = e.u;
  }
  std::vector<double> b(n);
  std::vector<int32_t> w_via(n), dep(n);
  for (int64_t v = 0; v < n; ++v) {  // every edge goes forward in stream order: ids are a topological order
    int32_t* p0 = pred.data() + off[v];
    int32_t* p1 = pred.data() + off[v + 1];
    std::sort(p0, p1);
    const bool copy = table[v * TINV_TASK_FIELDS + F_KIND] == TINV_COPY;
    const double w = weight ? weight[v] : (copy ? 0.0 : 1.0);
    double bb = 0.0;
    int32_t who = -1, dd = 0;
    for (int32_t* q = p0; q < p1; ++q) {
      if (q > p0 && *q == q[-1]) continue;
      if (b[*q] > bb) {  // strict: the smallest id wins a tie
        bb = b[*q];
        who = *q;
      }
      dd = std::max(dd, dep[*q]);
    }
    b[v] = bb + w;
    w_via[v] = who;
    dep[v] = dd + 1;
  }
  if (best) std::copy(b.begin(), b.end(), best);
  if (via) std::copy(w_via.begin(), w_via.end(), via);
  if (depth) std::copy(dep.begin(), dep.end(), depth);
  if (ncomp) {  // union-find over the kept tasks
    std::vector<int32_t> root(n);
    std::vector<char> keep(n);
    for (int64_t v = 0; v < n; ++v) {
      root[v] = (int32_t)v;
      keep[v] = include_copies || table[v * TINV_TASK_FIELDS + F_KIND] != TINV_COPY;
    }
    auto find = [&](int32_t x) {
      while (root[x] != x) x = root[x] = root[root[x]];
      return x;
    };
    for (const Edge& e : edges)
      if (keep[e.u] && keep[e.v]) {
        const int32_t ru = find(e.u), rv = find(e.v);
        if (ru != rv) root[ru] = rv;
      }
    int64_t c = 0;
    for (int64_t v = 0; v < n; ++v) c += keep[v] && find((int32_t)v) == v;
    *ncomp = c;
  }
  return TINV_OK;
}

int tinv_dist_stream(const int32_t* table, int64_t n, int32_t t, int32_t P, int32_t Q, int32_t* out, int64_t cap,
                     int64_t* nout, int32_t* owner, int32_t* dest, int32_t* ref) {
  if ((!table && n > 0) || t < 1 || P < 1 || Q < 1 || P * Q > 64)
    return fail(nullptr, TINV_ERR_BAD_ARG, "bad dist_stream arguments");
  auto own = [&](int r, int c) { return (r % P) * Q + (c % Q); };
  auto key = [&](const int32_t* f, int which) -> int64_t {  // which: 0 out, 1 r0, 2 r1
    const int o = which == 0 ? F_OL : (which == 1 ? F_R0L : F_R1L);
    return tile_key(f[o], f[o + 1], f[o + 2]);
  };
  // pass 1: consumer ranks of every (tile, version), version = writer task (-1: initial)
  std::unordered_map<int64_t, int32_t> last;
  // (tile key, version) pairs are exact keys: an ordered map on the pair (no
  // hashing into one int64, which could merge two versions' rank masks)
  typedef std::pair<int64_t, int32_t> VKey;
  std::map<VKey, uint64_t> need;   // (tile key, version) -> rank mask
  std::vector<int64_t> init_order;  // tiles whose initial version travels, first-use order
  auto vkey = [](int64_t tk, int32_t ver) { return VKey(tk, ver); };
  std::map<VKey, std::pair<int64_t, int32_t>> vinfo;  // vkey -> (tile key, version)
  for (int64_t v = 0; v < n; ++v) {
    const int32_t* f = table + v * TINV_TASK_FIELDS;
    const int rv = own(f[F_OR], f[F_OC]);
    for (int x = 0; x < f[F_NR] && x < 2; ++x) {
      const int o = x == 0 ? F_R0L : F_R1L;
      if (own(f[o + 1], f[o + 2]) == rv) continue;
      const int64_t tk = key(f, x + 1);
      auto it = last.find(tk);
      const int32_t ver = it == last.end() ? -1 : it->second;
      const VKey vk = vkey(tk, ver);
      if (!vinfo.count(vk)) {
        vinfo[vk] = {tk, ver};
        if (ver < 0) init_order.push_back(tk);
      }
      need[vk] |= 1ull << rv;
    }
    last[key(f, 0)] = (int32_t)v;
  }
  // pass 2: emit
  std::vector<Tk> res;
  std::vector<int32_t> ow, de, rf;
  std::map<std::pair<VKey, int>, int32_t> recv_label;  // (vkey, rank) -> label
  int32_t next_label = 64;
  std::unordered_map<int64_t, std::array<int32_t, 3>> tile_of;  // tile key -> (label, row, col)
  auto emit_sends = [&](int64_t tk, int32_t ver, int lab, int r, int c) {
    auto it = need.find(vkey(tk, ver));
    if (it == need.end()) return;
    for (int d = 0; d < 64; ++d)
      if (it->second >> d & 1) {
        const int32_t lbl = next_label++;
        recv_label[{vkey(tk, ver), d}] = lbl;
        Tk cp = {{TINV_COPY, TINV_STEP_COPY, r, c, -1, lbl, r, c, 2, 1, lab, r, c, -1, -1, -1}};
        res.push_back(cp);
        ow.push_back(own(r, c));
        de.push_back(d);
        rf.push_back(-1);
      }
  };
  for (int64_t v = 0; v < n; ++v) {  // tiles referenced, for the initial sends
    const int32_t* f = table + v * TINV_TASK_FIELDS;
    for (int x = 0; x < 3; ++x) {
      const int o = x == 0 ? F_OL : (x == 1 ? F_R0L : F_R1L);
      if (x > 0 && f[F_NR] < x) continue;
      tile_of[tile_key(f[o], f[o + 1], f[o + 2])] = {f[o], f[o + 1], f[o + 2]};
    }
  }
  for (int64_t tk : init_order) {
    const auto& tl = tile_of[tk];
    emit_sends(tk, -1, tl[0], tl[1], tl[2]);
  }
  last.clear();
  for (int64_t v = 0; v < n; ++v) {
    Tk task;
    memcpy(task.f, table + v * TINV_TASK_FIELDS, sizeof(task.f));
    int32_t* f = task.f;
    const int rv = own(f[F_OR], f[F_OC]);
    for (int x = 0; x < f[F_NR] && x < 2; ++x) {
      const int o = x == 0 ? F_R0L : F_R1L;
      if (own(f[o + 1], f[o + 2]) == rv) continue;
      const int64_t tk = tile_key(f[o], f[o + 1], f[o + 2]);
      auto it = last.find(tk);
      const int32_t ver = it == last.end() ? -1 : it->second;
      const auto rl = recv_label.find({vkey(tk, ver), rv});
      if (rl == recv_label.end()) return fail(nullptr, TINV_ERR_INTERNAL, "dist_stream: missing receive label");
      f[o] = rl->second;
    }
    res.push_back(task);
    ow.push_back(rv);
    de.push_back(-1);
    rf.push_back((int32_t)v);
    const int64_t otk = tile_key(f[F_OL], f[F_OR], f[F_OC]);
    last[otk] = (int32_t)v;
    emit_sends(otk, (int32_t)v, f[F_OL], f[F_OR], f[F_OC]);
  }
  if (nout) *nout = (int64_t)res.size();
  if (out) {
    if (cap < (int64_t)res.size()) return fail(nullptr, TINV_ERR_BAD_ARG, "dist_stream capacity too small");
    memcpy(out, res.data(), res.size() * sizeof(Tk));
    memcpy(owner, ow.data(), ow.size() * 4);
    memcpy(dest, de.data(), de.size() * 4);
    memcpy(ref, rf.data(), rf.size() * 4);
  }
  return TINV_OK;
}

int tinv_plan_destroy(tinv_plan* p) {
  if (!p) return TINV_OK;
  if (p->d_tasks) cudaSetDevice(p->ctx->device);
  void* ptrs[] = {p->d_tasks, p->d_succ, p->d_indeg, p->d_done, p->d_cur,      p->d_alt,       p->d_queue, p->d_head,
                  p->d_tail,  p->d_ctr,  p->d_err,   p->d_progress, p->d_ts, p->d_te, p->d_tr, p->d_tsm, p->d_snap_from,
                  p->d_snap_to, p->d_phase, p->d_recv_task, p->d_inbox, p->d_depart_group, p->d_depart_count,
                  p->d_depart_seq, p->d_recv_gate, p->d_gate_flag, p->d_qoffs, p->d_idle};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  if (p->ev0) cudaEventDestroy(p->ev0);
  if (p->ev1) cudaEventDestroy(p->ev1);
  delete p;
  return TINV_OK;
}

static void set_err(tinv_err* err, int32_t task, int32_t kind, int32_t code, int32_t index) {
  if (!err) return;
  err->task_id = task;
  err->kind = kind;
  err->code = code;
  err->index = index;
}

}  // extern "C"


// aux (n x 2, or null): per-task (dest rank, receive sequence) of transfer
// pseudo-tasks (KIND_SEND / KIND_RECV, allowed only when aux is given);
// nrecv: inbox length (receive tiles pinned at slots 2T + seq).
// rank_of (n, or null) / nranks: ranks emulated in one launch -- task v runs
// on the CTAs of rank rank_of[v] (tasks the planner inserts for v inherit it).
namespace {
struct XTouch {  // per exec task: the logical tiles it reads and writes, and whether its output is renamed
  int32_t in0, in1, out;
  bool renamed;
};
}  // namespace

// does kind `k` write its output to the alternate (renamed) slot? (same rule as the item / priority loop)
static bool renames(int kind, bool alias) {
  return kind == TINV_TRMM_LEFT || kind == TINV_TRMM_RIGHT_NEG || kind == TINV_TRMM_LEFT_T || kind == TINV_LAUUM ||
         kind == TINV_TRSM || kind == TINV_TRTRI ||
         (alias && (kind == TINV_GEMM || kind == TINV_SYRK_SUB || kind == TINV_SYRK_ADD_T));
}

template <class XS>
static std::vector<XTouch> xs_touch(const XS& xs, int64_t nx) {
  std::vector<XTouch> v(nx);
  for (int64_t u = 0; u < nx; ++u)
    v[u] = {xs[u].in0, xs[u].in1, xs[u].out, renames(xs[u].kind, xs[u].in0 == xs[u].out || xs[u].in1 == xs[u].out)};
  return v;
}

// Memory-constrained renaming (PAPER.md's closing open problem: performance
// under a memory constraint). Working tiles (the B / C copies of the
// out-of-place placement, INV and POTRF aux tiles) get slots by interval
// coloring over their live ranges in stream order -- [first task that touches
// the tile, last one] -- instead of one slot (pair) each. A tile that takes
// over a slot group gets edges from every task that touched the previous
// occupant to its first writer, so the reuse is safe under ANY schedule the
// executor picks (all those tasks precede it in stream order: the DAG stays
// acyclic). Out-of-place, B dies within step 2 and C is born in step 3, so
// C reuses B's slots: the store shrinks from 4T to 3T tiles.
template <class XS>
static void share_slots_pass(const std::vector<XTouch>& tv, int64_t T, int64_t nlogical,
                             const std::unordered_map<int32_t, int32_t>& pinned, const XS& xs,
                             std::vector<int32_t>& group, std::vector<int32_t>& width, std::vector<Edge>& edges) {
  (void)xs;
  const int64_t nw = nlogical - T;
  std::vector<int64_t> first(nw, -1), last(nw, -1);
  std::vector<char> ren(nw, 0);
  std::vector<std::vector<int32_t>> touch(nw);
  auto see = [&](int32_t l, int64_t u) {
    if (l < T) return;
    const int64_t w = l - T;
    if (first[w] < 0) first[w] = u;
    last[w] = u;
    if (touch[w].empty() || touch[w].back() != (int32_t)u) touch[w].push_back((int32_t)u);
  };
  for (int64_t u = 0; u < (int64_t)tv.size(); ++u) {
    see(tv[u].in0, u);
    see(tv[u].in1, u);
    see(tv[u].out, u);
    if (tv[u].out >= T && tv[u].renamed) ren[tv[u].out - T] = 1;
  }
  group.assign(nw, -1);
  width.clear();
  std::vector<int64_t> order;
  for (int64_t w = 0; w < nw; ++w)
    if (first[w] >= 0 && !pinned.count((int32_t)(w + T))) order.push_back(w);
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return first[a] < first[b]; });
  // free groups per width: min-heap on the stream position their occupant was last touched
  typedef std::pair<int64_t, int32_t> Fr;  // (last touch, group)
  std::priority_queue<Fr, std::vector<Fr>, std::greater<Fr>> freeq[2];
  std::vector<int64_t> occupant;  // group -> current working tile
  std::priority_queue<Fr, std::vector<Fr>, std::greater<Fr>> busy[2];  // (last touch, group) of live occupants
  for (int64_t w : order) {
    const int k = ren[w] ? 1 : 0;
    while (!busy[k].empty() && busy[k].top().first < first[w]) {  // occupants dead before w is born
      freeq[k].push(busy[k].top());
      busy[k].pop();
    }
    int32_t g;
    if (!freeq[k].empty()) {
      g = freeq[k].top().second;
      freeq[k].pop();
      const int64_t prev = occupant[g];
      for (int32_t u : touch[prev]) edges.push_back({u, (int32_t)first[w], 1});  // slot reuse: WAR on the slot
      occupant[g] = w;
    } else {
      g = (int32_t)width.size();
      width.push_back(k ? 2 : 1);
      occupant.push_back(w);
    }
    group[w] = g;
    busy[k].push({last[w], g});
  }
}

int plan_build(tinv_ctx* c, const int32_t* table, int64_t n, int32_t stream_t, const int64_t* barriers,
               int64_t nbar, uint32_t flags, tinv_plan** out, tinv_err* err, const int32_t* aux, int64_t nrecv,
               const int32_t* rank_of, int32_t nranks, bool host_only) {
  set_err(err, -1, -1, TINV_OK, -1);
  if (!c || !out || (!table && n > 0)) return fail(c, TINV_ERR_BAD_ARG, "bad plan arguments");
  if (nranks < 1 || nranks > MAX_RANKS || (nranks > 1 && !rank_of) || nranks > c->nsm)
    return fail(c, TINV_ERR_BAD_ARG, "bad rank count");
  *out = nullptr;
  // scheduler.py:274-276
  if (stream_t != c->t) {
    set_err(err, -1, -1, TINV_ERR_STREAM, -1);
    return fail(c, TINV_ERR_STREAM, "stream generated for t=" + std::to_string(stream_t) +
                                        " cannot run on a t=" + std::to_string(c->t) + " matrix");
  }
  if (c->partitioned && (flags & (TINV_KEEP_ON_FAILURE | TINV_STREAM_IO)))
    return fail(c, TINV_ERR_BAD_ARG, "a partitioned store supports neither TINV_KEEP_ON_FAILURE nor TINV_STREAM_IO");
  const int R = (int)c->R, t = (int)c->t;
  const int64_t T = c->T;
  tinv_plan* p = new tinv_plan();
  p->ctx = c;
  p->flags = flags;
  p->nranks = nranks;

  // ---- logical tiles, validation, INV insertion for TRSM (renamed inverse)
  std::unordered_map<int64_t, int32_t> logical;  // key -> logical id (non-matrix tiles)
  std::vector<char> written_dyn;                 // per non-matrix logical: written so far
  int64_t next_logical = T;
  int64_t mm = 0;  // matrix of a batched store the task is replicated for
  const int64_t nm = c->nmat;  // batched store: the stream is replicated per matrix (no cross edges)
  auto get_logical = [&](int label, int r, int cc, bool is_read, int64_t task, int32_t& id) -> bool {
    if (label == 0) {
      if (r < 0 || r >= t || cc < 0 || cc > r) return false;
      id = (int32_t)(mm * c->T1 + tri_index(r, cc));
      return true;
    }
    if (label < 0 || label >= (nm > 1 ? (1 << 14) : (1 << 26)) || r < 0 || r >= t || cc < 0 || cc >= t) return false;
    const int64_t key = tile_key((int)(mm * (1 << 14) + label), r, cc);  // < 2^27 labels x 2^18 x 2^18
    auto it = logical.find(key);
    if (it == logical.end()) {
      if (is_read) return false;  // reference: store KeyError (never written)
      id = (int32_t)next_logical++;
      logical[key] = id;
      written_dyn.push_back(0);
    } else {
      id = it->second;
    }
    (void)task;
    return true;
  };
  std::vector<int32_t> last_writer_exec;  // per logical tile: exec index of last writer (-1 initial)
  last_writer_exec.assign(T, -1);
  std::unordered_map<int64_t, int32_t> inv_cache;  // (L logical << 32 | version+1) -> aux logical
  struct XT {
    int kind, step, out, in0, in1, mode, ref, aux0, aux1, flags;
  };
  std::unordered_map<int32_t, int32_t> recv_pin;  // receive tile -> sequence number
  if (nm > 1 && barriers && nbar > 0) {
    tinv_plan_destroy(p);
    return fail(c, TINV_ERR_BAD_ARG, "barriers are not supported on a batched store");
  }
  const bool sio = (flags & TINV_STREAM_IO) != 0;
  if (sio && (aux || (flags & TINV_KEEP_ON_FAILURE))) {
    tinv_plan_destroy(p);
    return fail(c, TINV_ERR_BAD_ARG, "streamed host I/O excludes transfer plans and TINV_KEEP_ON_FAILURE");
  }
  p->nref = n * nm;
  p->ref_kind.resize(n * nm);
  std::vector<XT> xs;
  xs.reserve(nm * (n + n / 8 + 8 + (sio ? 2 * c->T1 : 0)));
  if (sio) {  // ARRIVE: every lower tile of every matrix, column order (the order step 1 consumes them)
    for (int64_t m = 0; m < nm; ++m)
      for (int j = 0; j < t; ++j)
        for (int i = j; i < t; ++i) {
          const int32_t o = (int32_t)(m * c->T1 + tri_index(i, j));
          const int32_t seq = (int32_t)p->arrive_tile.size();
          last_writer_exec[o] = (int32_t)xs.size();
          xs.push_back({KIND_ARRIVE, 0, o, -1, -1, 2, -1, -1, seq, 0});
          p->arrive_tile.push_back(o);
        }
    nrecv = (int64_t)p->arrive_tile.size();
  }
  std::vector<char> is_aux;
  std::vector<int32_t> first_exec_of_ref(n * nm + 1, 0);
  std::vector<int8_t> xrank;  // rank of every exec task
  int8_t cur_rank = 0;
  for (int64_t rv = 0; rv < n * nm; ++rv) {
    while (xrank.size() < xs.size()) xrank.push_back(cur_rank);  // tasks made for the previous ref task
    cur_rank = rank_of ? (int8_t)rank_of[rv % n] : 0;
    if (cur_rank < 0 || cur_rank >= nranks) {
      tinv_plan_destroy(p);
      return fail(c, TINV_ERR_BAD_ARG, "task rank out of range");
    }
    mm = rv / n;
    const int64_t v = rv;
    const int32_t* f = table + (rv % n) * TINV_TASK_FIELDS;
    const int kind = f[F_KIND];
    p->ref_kind[v] = kind;
    first_exec_of_ref[v] = (int32_t)xs.size();
    auto bad = [&](const std::string& why) {
      set_err(err, (int32_t)v, kind, TINV_ERR_STREAM, -1);
      tinv_plan_destroy(p);
      return fail(c, TINV_ERR_STREAM, "task " + std::to_string(v) + ": " + why);
    };
    const bool xfer = aux && (kind == KIND_SEND || kind == KIND_RECV);
    if ((kind < TINV_COPY || kind > TINV_LAUUM) && !xfer) return bad("unknown kernel kind");
    if (kind == TINV_GEMM && (f[F_STEP] < 1 || f[F_STEP] > 3)) return bad("unsupported gemm shape");
    const int nr = f[F_NR];
    if (nr != expected_reads(kind)) return bad("wrong number of operands");
    int32_t in0 = -1, in1 = -1, o = -1;
    if (nr >= 1 && !get_logical(f[F_R0L], f[F_R0R], f[F_R0C], true, v, in0)) return bad("read of a missing tile");
    if (nr >= 2 && !get_logical(f[F_R1L], f[F_R1R], f[F_R1C], true, v, in1)) return bad("read of a missing tile");
    const int32_t ax0 = aux ? aux[2 * (rv % n)] : -1, ax1 = aux ? aux[2 * (rv % n) + 1] : -1;
    if (kind == KIND_SEND) {  // reads its tile version, writes nothing locally
      xs.push_back({kind, 0, -1, in0, -1, 0, (int)v, ax0, ax1, 0});
      continue;
    }
    if (!get_logical(f[F_OL], f[F_OR], f[F_OC], false, v, o)) return bad("output tile outside the matrix");
    if (c->partitioned)
      for (int32_t tl : {in0, in1, o})
        if (tl >= 0 && tl < T && c->home[tl] < 0) return bad("tile of another rank's store (partitioned context)");
    if (kind == KIND_RECV) {
      if (ax1 < 0 || ax1 >= nrecv) return bad("receive sequence out of range");
      recv_pin[o] = ax1;
      written_dyn[o - T] = 1;
      if ((int64_t)last_writer_exec.size() < next_logical) last_writer_exec.resize(next_logical, -1);
      last_writer_exec[o] = (int32_t)xs.size();
      xs.push_back({kind, 0, o, -1, -1, 2, (int)v, ax0, ax1, 0});
      continue;
    }
    if (kind != TINV_COPY && f[F_OL] != 0 && o >= T && !written_dyn[o - T]) return bad("kernel on an unwritten tile");
    if ((int64_t)last_writer_exec.size() < next_logical) last_writer_exec.resize(next_logical, -1);
    int xflags = 0;
    // the factor's diagonal-block inverses computed by POTRF (its aux tile)
    auto potrf_aux = [&](int32_t tile) -> int32_t {
      const int32_t w = last_writer_exec[tile];
      return (w >= 0 && (xs[w].kind == TINV_POTRF || xs[w].kind == KIND_POTRF_INV)) ? xs[w].in0 : -1;
    };
    auto full_inv_aux = [&](int32_t tile) -> int32_t {  // aux of a POTRF_INV (full inverse) or -1
      const int32_t w = last_writer_exec[tile];
      return (w >= 0 && xs[w].kind == KIND_POTRF_INV) ? xs[w].in0 : -1;
    };
    if (kind == TINV_TRTRI) {  // TRTRI of an unchanged factor: copy POTRF_INV's inverse, or reuse INV's,
                               // or start from POTRF's diagonal-block inverses
      int32_t src_inv = full_inv_aux(o);
      if (src_inv < 0) {
        const int64_t key = ((int64_t)o << 32) | (int64_t)(last_writer_exec[o] + 1);
        auto it = inv_cache.find(key);
        if (it != inv_cache.end()) src_inv = it->second;
      }
      if (src_inv >= 0) {
        last_writer_exec[o] = (int32_t)xs.size();
        xs.push_back({TINV_COPY, TINV_STEP_COPY, o, src_inv, -1, 1, (int)v, -1, -1, 0});
        continue;
      }
      const int32_t pa = potrf_aux(o);
      if (pa >= 0) {
        in1 = pa;
        xflags = TF_DIAG_FROM_AUX;
      }
    }
    if (kind == TINV_TRSM && potrf_aux(in0) >= 0) {
      // multiply by the factor's inverse, kept whole by the POTRF (no INV task on the critical path)
      xs[last_writer_exec[in0]].kind = KIND_POTRF_INV;
      in0 = potrf_aux(in0);
    } else if (kind == TINV_TRSM) {
      const int64_t key = ((int64_t)in0 << 32) | (int64_t)(last_writer_exec[in0] + 1);
      auto it = inv_cache.find(key);
      int32_t inv_t;
      if (it == inv_cache.end()) {
        inv_t = (int32_t)next_logical++;
        written_dyn.push_back(1);
        is_aux.resize(next_logical - T, 0);
        is_aux[inv_t - T] = 1;
        last_writer_exec.resize(next_logical, -1);
        last_writer_exec[inv_t] = (int32_t)xs.size();
        const int32_t pa = potrf_aux(in0);
        xs.push_back({KIND_INV, f[F_STEP], inv_t, in0, pa, 1, (int)v, -1, -1, pa >= 0 ? TF_DIAG_FROM_AUX : 0});
        inv_cache[key] = inv_t;
      } else {
        inv_t = it->second;
      }
      in0 = inv_t;
    }
    if (kind == TINV_POTRF) {  // private aux tile: inverses of the diagonal blocks of L
      in0 = (int32_t)next_logical++;
      written_dyn.push_back(1);
      last_writer_exec.resize(next_logical, -1);
    }
    if (o >= T) written_dyn[o - T] = 1;
    last_writer_exec[o] = (int32_t)xs.size();
    xs.push_back({kind, f[F_STEP], o, in0, in1, f[F_OM] == 2 ? 2 : 1, (int)v, -1, -1, xflags});
  }
  first_exec_of_ref[n * nm] = (int32_t)xs.size();
  while (xrank.size() < xs.size()) xrank.push_back(cur_rank);
  std::vector<int32_t> depart_lw;  // last writer of each departing tile
  if (sio)  // DEPART: every lower tile of every matrix, after its last writer
    for (int64_t m = 0; m < nm; ++m)
      for (int i = 0; i < t; ++i)
        for (int j = 0; j <= i; ++j) {
          const int32_t o = (int32_t)(m * c->T1 + tri_index(i, j));
          depart_lw.push_back(last_writer_exec[o]);
          p->depart_tile.push_back(o);
          xs.push_back({KIND_DEPART, 0, -1, o, -1, 0, -1, o, (i << 16) | j, 0});
        }
  p->nexec = (int64_t)xs.size();
  p->nlogical = next_logical;
  const int64_t nx = p->nexec;
  // SYRK_SUB whose tile is next written by a POTRF, through SYRK_SUBs only
  // (step 1's trailing diagonal chain): POTRF reads the lower triangle and
  // zeroes the rest, so its strict upper part is dead -- the task reduce-adds
  // its lower blocks with the TMA epilogue instead of mirroring through the
  // generic one (C2: SYRK_SUB 60 -> ~40 us on the critical path).
  {
    std::vector<std::vector<int32_t>> users(next_logical);
    for (int64_t u = 0; u < nx; ++u)
      for (int32_t tl : {xs[u].in0, xs[u].in1, xs[u].out})
        if (tl >= 0 && (users[tl].empty() || users[tl].back() != (int32_t)u)) users[tl].push_back((int32_t)u);
    for (int64_t u = 0; u < nx; ++u) {
      if (xs[u].kind != TINV_SYRK_SUB || xs[u].in0 == xs[u].out || xs[u].in1 == xs[u].out) continue;
      const auto& us = users[xs[u].out];
      auto it = std::upper_bound(us.begin(), us.end(), (int32_t)u);
      bool dead = false;
      for (; it != us.end(); ++it) {
        const auto& w = xs[*it];
        if (w.kind == TINV_SYRK_SUB && w.out == xs[u].out && w.in0 != w.out && w.in1 != w.out) continue;
        dead = (w.kind == TINV_POTRF || w.kind == KIND_POTRF_INV) && w.out == xs[u].out;
        break;
      }
      if (dead) xs[u].flags |= TF_NO_MIRROR;
    }
  }

  // ---- memory-constrained renaming (TINV_SHARE_SLOTS): working tiles share slots
  std::vector<int32_t> share_group;  // non-matrix logical tile - T -> slot group (-1: own slots)
  std::vector<int32_t> share_width;  // slots per group (1, or 2 for a renamed tile's cur / alt pair)
  // ---- hazard DAG over exec tasks (+ barrier edges at translated positions)
  {
    std::vector<std::vector<Acc>> acc(nx);
    for (int64_t v = 0; v < nx; ++v) {
      const bool potrf = xs[v].kind == TINV_POTRF || xs[v].kind == KIND_POTRF_INV;
      if (xs[v].in0 >= 0 && !potrf) acc[v].push_back({xs[v].in0, 0});
      if (xs[v].in0 >= 0 && potrf) acc[v].push_back({xs[v].in0, 2});  // writes its aux
      if (xs[v].in1 >= 0) acc[v].push_back({xs[v].in1, 0});
      if (xs[v].out >= 0) acc[v].push_back({xs[v].out, xs[v].mode});
    }
    std::vector<int64_t> bars;
    for (int64_t x = 0; x < (barriers ? nbar : 0); ++x) {
      const int64_t pos = barriers[x];
      if (pos < 0 || pos > n) {
        tinv_plan_destroy(p);
        return fail(c, TINV_ERR_STREAM, "barrier position out of range");
      }
      bars.push_back(first_exec_of_ref[pos]);
    }
    std::vector<Edge> edges;
    scoreboard(nx, acc, bars, edges);
    if (flags & TINV_SERIAL)
      for (int64_t v = 0; v + 1 < nx; ++v) edges.push_back({(int32_t)v, (int32_t)(v + 1), 3});
    if (flags & TINV_SHARE_SLOTS) share_slots_pass(xs_touch(xs, nx), T, next_logical, recv_pin, xs, share_group,
                                                   share_width, edges);
    std::vector<std::vector<int32_t>> adj(nx);
    for (const Edge& e : edges) adj[e.u].push_back(e.v);
    p->indeg0.assign(nx, 0);
    p->tasks.resize(nx);
    int64_t ne = 0;
    for (int64_t u = 0; u < nx; ++u) {
      auto& a = adj[u];
      std::sort(a.begin(), a.end());
      a.erase(std::unique(a.begin(), a.end()), a.end());
      p->tasks[u].succ_begin = (int32_t)p->succ.size();
      for (int32_t v : a) {
        p->succ.push_back(v);
        p->indeg0[v]++;
      }
      p->tasks[u].succ_end = (int32_t)p->succ.size();
      ne += (int64_t)a.size();
    }
    p->nedges = ne;
  }

  // ---- items, renaming, priorities (bottom level in estimated critical-path time)
  std::vector<double> bl(nx, 0.0);
  double blmax = 0.0;
  // streamed output: a departure weighs like `dw` b^3 of work, pulling the
  // chains that finish result tiles forward so the copy engines overlap them
  const char* dws = getenv("TINV_DEPART_WEIGHT");
  const double dw = dws ? atof(dws) : kDepartWeight;
  // bottom levels in estimated critical-path time (latency_of; TINV_PRIO=flops: in flops).
  // Measured: C2 20.94 -> 20.41 ms, C3 1034.5 -> 1031.6 ms, C1 unchanged.
  const char* pr = getenv("TINV_PRIO");
  const bool lat = !(pr && !strcmp(pr, "flops"));
  // level = floor(NLEV (1 - (bl / blmax)^e)): e < 1 spends more of the 32
  // levels on the short remaining paths of the DAG's tail, where a critical
  // chain (C2: the SYRK_ADD_T chain of step 3) otherwise queues FIFO behind
  // hundreds of same-level items. Measured e = 1 / 0.3 / 0.1: C2 20.4 / 20.1 /
  // 19.5 ms, C3 and C4 (DAG) unchanged. Streamed plans keep e = 1: the
  // compressed curve defers the chains that finish result tiles, so the
  // device -> host copies pile up at the end (C3 e2e 1062 -> 1218 ms).
  // TINV_PRIO_EXP overrides both.
  const char* pe = getenv("TINV_PRIO_EXP");
  // Transfer plans (multi-GPU, aux given) use e = 10: resolution at the TOP
  // of the bottom-level range, where the distributed run is critical-path
  // bound (the step-1 panel chain crossing ranks through SEND / RECV). In the
  // schedule model (csrc/model.cu, tools/scaling_model.py) at C3 on 8 B200s:
  // e = 0.1 / 1 / 4 / 10 -> 235 / 232 / 181 / 150 ms (efficiency 0.54 ->
  // 0.84), the one-launch emulation on one B200 agreeing with the model.
  const double prio_exp = pe ? std::max(0.01, atof(pe)) : (sio ? 1.0 : (aux ? 10.0 : 0.1));
  for (int64_t u = nx - 1; u >= 0; --u) {
    double m = 0.0;
    for (int32_t k = p->tasks[u].succ_begin; k < p->tasks[u].succ_end; ++k) m = std::max(m, bl[p->succ[k]]);
    bl[u] = (xs[u].kind == KIND_DEPART ? dw : lat ? latency_of(xs[u].kind, R, xs[u].flags) : weight_of(xs[u].kind)) + m;
    blmax = std::max(blmax, bl[u]);
  }
  std::vector<char> renamed_tile(p->nlogical, 0);
  if (sio) p->rename_parity.assign(T, 0);
  const int NQ = nranks * NLEV;  // queue sets: one per rank
  std::vector<int64_t> lev_items(NQ, 0);

  FILE* dump = getenv("TINV_DUMP_LEVELS") ? fopen(getenv("TINV_DUMP_LEVELS"), "w") : nullptr;  // debug
  p->exec_ref.resize(nx);
  for (int64_t u = 0; u < nx; ++u) {
    TaskDev& d = p->tasks[u];
    const XT& x = xs[u];
    d.kind = (int8_t)x.kind;
    d.step = (int8_t)x.step;
    d.out = x.out;
    d.in0 = x.in0;
    d.in1 = x.in1;
    d.ref_id = x.ref;
    d.aux0 = x.aux0;
    d.aux1 = x.aux1;
    d.nitems = total_items(x.kind, R);
    d.nphases = (int16_t)ngroups(x.kind, R);
    d.rank = u < (int64_t)xrank.size() ? xrank[u] : 0;  // DEPART (streamed plans, one rank): 0
    d.pad = 0;
    d.flags = (int8_t)x.flags;
    const bool alias = (x.in0 == x.out || x.in1 == x.out);
    if (x.kind == TINV_TRMM_LEFT || x.kind == TINV_TRMM_RIGHT_NEG || x.kind == TINV_TRMM_LEFT_T ||
        x.kind == TINV_LAUUM || x.kind == TINV_TRSM || x.kind == TINV_TRTRI ||
        (alias && (x.kind == TINV_GEMM || x.kind == TINV_SYRK_SUB || x.kind == TINV_SYRK_ADD_T))) {
      d.flags |= TF_RENAMED;
      renamed_tile[x.out] = 1;
      if (sio && x.out < T) p->rename_parity[x.out] ^= 1;
    }
    if (x.kind == KIND_RECV || x.kind == KIND_ARRIVE) d.flags |= TF_EXTERNAL;
    int lev = blmax > 0 ? (int)std::floor(NLEV * (1.0 - std::pow(bl[u] / blmax, prio_exp))) : 0;
    lev = std::min(NLEV - 1, std::max(0, lev));
    if (x.kind == KIND_DEPART) lev = 0;  // cheap, and the copy engines wait on it
    if (dump) fprintf(dump, "%lld %d %d %d %.3f %d\n", (long long)u, x.kind, x.ref, x.out, bl[u], lev);
    d.level = (int8_t)lev;
    lev_items[d.rank * NLEV + lev] += d.nitems;
    p->items += d.nitems;
    p->exec_ref[u] = x.ref;
  }
  if (dump) fclose(dump);
  if (sio) {  // departures in predicted completion order: the last writer's top level (earliest finish on
              // unbounded workers); after a run the observed order replaces it (tinv_plan_exec_host)
    std::vector<double> tl(nx, 0.0);
    for (int64_t u = 0; u < nx; ++u) {
      tl[u] += weight_of(xs[u].kind);
      for (int32_t k = p->tasks[u].succ_begin; k < p->tasks[u].succ_end; ++k)
        tl[p->succ[k]] = std::max(tl[p->succ[k]], tl[u]);
    }
    std::vector<int32_t> ord(p->depart_tile.size());
    for (size_t k = 0; k < ord.size(); ++k) ord[k] = (int32_t)k;
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) {
      const double ax = depart_lw[x] >= 0 ? tl[depart_lw[x]] : 0.0, ay = depart_lw[y] >= 0 ? tl[depart_lw[y]] : 0.0;
      return ax < ay;
    });
    std::vector<int32_t> dt(ord.size());
    for (size_t k = 0; k < ord.size(); ++k) dt[k] = p->depart_tile[ord[k]];
    p->depart_tile.swap(dt);
  }
  p->q_off.assign(NQ + 1, 0);
  for (int l = 0; l < NQ; ++l) p->q_off[l + 1] = p->q_off[l] + lev_items[l];
  p->tail0.assign(NQ, 0);
  p->q_init.assign(p->q_off[NQ], 0ull);
  for (int64_t u = 0; u < nx; ++u)
    if (p->indeg0[u] == 0 && !(p->tasks[u].flags & TF_EXTERNAL)) {
      const TaskDev& d = p->tasks[u];
      const int q = d.rank * NLEV + d.level;
      for (int i = 0; i < group_items(d.kind, R, 0); ++i)
        p->q_init[p->q_off[q] + p->tail0[q]++] = ((unsigned long long)(u + 1) << 32) | (unsigned)i;
    }

  // ---- slots of the non-matrix logical tiles: [2T, 2T + dyn)
  p->cur0.assign(p->nlogical, -1);
  p->alt0.assign(p->nlogical, -1);
  const int64_t mslots = c->mslots;
  int64_t next_slot = mslots + nrecv;  // receive tiles pinned at mslots + seq
  std::vector<int32_t> group_slot(share_width.size(), -1);
  for (int64_t l = T; l < p->nlogical; ++l) {
    auto pin = recv_pin.find((int32_t)l);
    if (pin != recv_pin.end()) {
      p->cur0[l] = p->alt0[l] = (int32_t)(mslots + pin->second);
      continue;
    }
    const int32_t gr = l - T < (int64_t)share_group.size() ? share_group[l - T] : -1;
    if (gr >= 0) {  // a slot group shared by working tiles with disjoint live ranges
      if (group_slot[gr] < 0) {
        group_slot[gr] = (int32_t)next_slot;
        next_slot += share_width[gr];
      }
      p->cur0[l] = group_slot[gr];
      p->alt0[l] = renamed_tile[l] ? group_slot[gr] + 1 : p->cur0[l];
      continue;
    }
    p->cur0[l] = (int32_t)next_slot++;
    p->alt0[l] = renamed_tile[l] ? (int32_t)next_slot++ : p->cur0[l];
  }
  p->dyn_slots = next_slot - mslots;
  p->nrecv = nrecv;
  p->recv_task_h.assign(std::max<int64_t>(nrecv, 1), -1);
  for (int64_t u = 0; u < nx; ++u)
    if (xs[u].kind == KIND_RECV || xs[u].kind == KIND_ARRIVE) p->recv_task_h[xs[u].aux1] = (int32_t)u;

  if (host_only) {  // schedule model: the compiled DAG only
    *out = p;
    return TINV_OK;
  }
  // ---- device buffers
  auto ckm = [&](void** ptr, size_t bytes) { return cudaMalloc(ptr, std::max<size_t>(bytes, 16)); };
  if (cudaSetDevice(c->device) != cudaSuccess || ckm((void**)&p->d_tasks, nx * sizeof(TaskDev)) ||
      ckm((void**)&p->d_succ, p->succ.size() * 4) || ckm((void**)&p->d_indeg, nx * 4) ||
      ckm((void**)&p->d_done, nx * 4) || ckm((void**)&p->d_cur, p->nlogical * 4) ||
      ckm((void**)&p->d_alt, p->nlogical * 4) || ckm((void**)&p->d_queue, p->q_off[NQ] * 8) ||
      ckm((void**)&p->d_head, NQ * 4) || ckm((void**)&p->d_tail, NQ * 4) || ckm((void**)&p->d_ctr, 2 * 4) ||
      ckm((void**)&p->d_qoffs, (NQ + 1) * 8) || ckm((void**)&p->d_idle, (size_t)c->nsm * 8) ||
      ckm((void**)&p->d_err, 8) || ckm((void**)&p->d_progress, 4) || cudaEventCreate(&p->ev0) ||
      cudaEventCreate(&p->ev1)) {
    tinv_plan_destroy(p);
    cudaGetLastError();
    return fail(c, TINV_ERR_CUDA, "plan allocation failed");
  }
  if (flags & TINV_TRACE) {
    if (ckm((void**)&p->d_ts, nx * 8) || ckm((void**)&p->d_te, nx * 8) || ckm((void**)&p->d_tsm, nx * 4) ||
        ckm((void**)&p->d_tr, 2 * nx * 8)) {
      tinv_plan_destroy(p);
      return fail(c, TINV_ERR_CUDA, "trace allocation failed");
    }
  }
  if (flags & TINV_KEEP_ON_FAILURE) {
    if (ckm((void**)&p->d_snap_from, T * 4) || ckm((void**)&p->d_snap_to, T * 4)) {
      tinv_plan_destroy(p);
      return fail(c, TINV_ERR_CUDA, "snapshot allocation failed");
    }
  }
  if (sio && (ckm((void**)&p->d_depart_group, T * 4) || ckm((void**)&p->d_depart_count, T * 4) ||
              ckm((void**)&p->d_depart_seq, (T + 1) * 4) || ckm((void**)&p->d_recv_gate, nrecv * 4) ||
              ckm((void**)&p->d_gate_flag, nrecv * 4))) {
    tinv_plan_destroy(p);
    return fail(c, TINV_ERR_CUDA, "departure counters allocation failed");
  }
  if (ckm((void**)&p->d_recv_task, p->recv_task_h.size() * 4) || ckm((void**)&p->d_inbox, p->recv_task_h.size() * 4)) {
    tinv_plan_destroy(p);
    return fail(c, TINV_ERR_CUDA, "inbox allocation failed");
  }
  cudaMemcpy(p->d_recv_task, p->recv_task_h.data(), p->recv_task_h.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(p->d_qoffs, p->q_off.data(), (NQ + 1) * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(p->d_tasks, p->tasks.data(), nx * sizeof(TaskDev), cudaMemcpyHostToDevice);
  if (!p->succ.empty()) cudaMemcpy(p->d_succ, p->succ.data(), p->succ.size() * 4, cudaMemcpyHostToDevice);
  if (cudaGetLastError() != cudaSuccess) {
    tinv_plan_destroy(p);
    return fail(c, TINV_ERR_CUDA, "plan upload failed");
  }
  *out = p;
  return TINV_OK;
}

extern "C" {

int tinv_plan_create(tinv_ctx* c, const int32_t* table, int64_t n, int32_t stream_t, const int64_t* barriers,
                     int64_t nbar, uint32_t flags, tinv_plan** out, tinv_err* err) {
  return plan_build(c, table, n, stream_t, barriers, nbar, flags, out, err, nullptr, 0, nullptr, 1, false);
}

int tinv_plan_create_xfer(tinv_ctx* c, const int32_t* table, int64_t n, int32_t stream_t, const int32_t* aux,
                          int64_t nrecv, uint32_t flags, tinv_plan** out, tinv_err* err) {
  if (!aux) return fail(c, TINV_ERR_BAD_ARG, "transfer plans need the aux table");
  return plan_build(c, table, n, stream_t, nullptr, 0, flags, out, err, aux, nrecv, nullptr, 1, false);
}

int tinv_plan_create_ranks(tinv_ctx* c, const int32_t* table, int64_t n, int32_t stream_t, const int32_t* aux,
                           int64_t nrecv, const int32_t* rank_of, int32_t nranks, uint32_t flags, tinv_plan** out,
                           tinv_err* err) {
  if (!aux || !rank_of) return fail(c, TINV_ERR_BAD_ARG, "rank plans need the aux and rank tables");
  if (flags & TINV_STREAM_IO) return fail(c, TINV_ERR_BAD_ARG, "rank plans exclude streamed host I/O");
  return plan_build(c, table, n, stream_t, nullptr, 0, flags, out, err, aux, nrecv, rank_of, nranks, false);
}

int tinv_plan_cta_idle(const tinv_plan* p, int64_t* idle_ns, int32_t* rank, int64_t cap, int64_t* nctas) {
  if (!p) return TINV_ERR_BAD_ARG;
  const int64_t g = (int64_t)p->h_idle.size();
  if (nctas) *nctas = g;
  if (idle_ns || rank) {
    if (cap < g) return fail(p->ctx, TINV_ERR_BAD_ARG, "cta_idle capacity too small");
    for (int64_t b = 0; b < g; ++b) {
      if (idle_ns) idle_ns[b] = (int64_t)p->h_idle[b];
      if (rank) rank[b] = (int32_t)(b % p->nranks);
    }
  }
  return TINV_OK;
}

int tinv_ipc_export(tinv_ctx* c, tinv_plan* p, void* pool_handle, void* inbox_handle) {
  if (!c || !p || !pool_handle || !inbox_handle) return fail(c, TINV_ERR_BAD_ARG, "bad ipc_export arguments");
  CK(c, cudaSetDevice(c->device));
  const int64_t need = c->mslots + p->dyn_slots + c->nsm + ((p->flags & TINV_KEEP_ON_FAILURE) ? c->T : 0);
  int rc = ensure_pool(c, need);
  if (rc) return rc;
  if (!c->inbox || c->inbox_len < std::max<int64_t>(p->nrecv, 1)) {
    if (c->exported) return fail(c, TINV_ERR_BAD_ARG, "inbox already exported");
    if (c->inbox) cudaFree(c->inbox);
    c->inbox_len = std::max<int64_t>(p->nrecv, 1);
    CK(c, cudaMalloc(&c->inbox, c->inbox_len * 4));
    CK(c, cudaMemset(c->inbox, 0, c->inbox_len * 4));
  }
  cudaIpcMemHandle_t hp, hi;
  CK(c, cudaIpcGetMemHandle(&hp, c->pool));
  CK(c, cudaIpcGetMemHandle(&hi, c->inbox));
  memcpy(pool_handle, &hp, sizeof(hp));
  memcpy(inbox_handle, &hi, sizeof(hi));
  c->exported = true;
  return TINV_OK;
}

int tinv_ipc_open(tinv_ctx* c, int32_t rank, int32_t world, const void* pool_handles, const void* inbox_handles) {
  if (!c || rank < 0 || world < 1 || world > MAX_RANKS || rank >= world || !pool_handles || !inbox_handles)
    return fail(c, TINV_ERR_BAD_ARG, "bad ipc_open arguments");
  if (!c->exported) return fail(c, TINV_ERR_BAD_ARG, "export this rank's store first");
  CK(c, cudaSetDevice(c->device));
  c->rank = rank;
  c->world = world;
  for (int r = 0; r < world; ++r) {
    if (r == rank) {
      c->peer_pool[r] = c->pool;
      c->peer_inbox[r] = c->inbox;
      continue;
    }
    cudaIpcMemHandle_t hp, hi;
    memcpy(&hp, (const char*)pool_handles + r * sizeof(hp), sizeof(hp));
    memcpy(&hi, (const char*)inbox_handles + r * sizeof(hi), sizeof(hi));
    void *pp = nullptr, *pi = nullptr;
    CK(c, cudaIpcOpenMemHandle(&pp, hp, cudaIpcMemLazyEnablePeerAccess));
    CK(c, cudaIpcOpenMemHandle(&pi, hi, cudaIpcMemLazyEnablePeerAccess));
    c->peer_pool[r] = (double*)pp;
    c->peer_inbox[r] = (int32_t*)pi;
  }
  return TINV_OK;
}

int tinv_peer_attach(tinv_ctx* c, int32_t rank, int32_t world, tinv_ctx* const* peers) {
  if (!c || !peers || rank < 0 || world < 1 || world > MAX_RANKS || rank >= world || peers[rank] != c)
    return fail(c, TINV_ERR_BAD_ARG, "bad peer_attach arguments");
  for (int r = 0; r < world; ++r)
    if (!peers[r] || !peers[r]->exported || peers[r]->device != c->device)
      return fail(c, TINV_ERR_BAD_ARG, "every peer must be exported, on this device");
  c->rank = rank;
  c->world = world;
  c->attached = true;  // plain pointers: nothing to close
  for (int r = 0; r < world; ++r) {
    c->peer_pool[r] = peers[r]->pool;
    c->peer_inbox[r] = peers[r]->inbox;
    c->peer_rbase[r] = (int32_t)peers[r]->mslots;
  }
  return TINV_OK;
}

int tinv_ipc_recv_bases(tinv_ctx* c, int32_t world, const int32_t* bases) {
  if (!c || !bases || world < 1 || world > MAX_RANKS) return fail(c, TINV_ERR_BAD_ARG, "bad ipc_recv_bases arguments");
  for (int r = 0; r < world; ++r) c->peer_rbase[r] = bases[r];
  return TINV_OK;
}

int tinv_recv_base(const tinv_ctx* c, int32_t* base) {
  if (!c || !base) return TINV_ERR_BAD_ARG;
  *base = (int32_t)c->mslots;
  return TINV_OK;
}

int tinv_set_sms(tinv_ctx* c, int32_t nsm) {
  if (!c) return TINV_ERR_BAD_ARG;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, c->device) != cudaSuccess) return fail(c, TINV_ERR_CUDA, "device query failed");
  if (nsm < 1 || nsm > prop.multiProcessorCount) return fail(c, TINV_ERR_BAD_ARG, "nsm out of range");
  c->nsm = nsm;
  return TINV_OK;
}

int tinv_ipc_reset(tinv_ctx* c) {
  if (!c || !c->inbox) return fail(c, TINV_ERR_BAD_ARG, "no exported inbox");
  CK(c, cudaSetDevice(c->device));
  CK(c, cudaMemset(c->inbox, 0, c->inbox_len * 4));
  CK(c, cudaDeviceSynchronize());
  return TINV_OK;
}

int tinv_plan_stats(const tinv_plan* p, int64_t* exec_tasks, int64_t* items, int64_t* edges) {
  if (!p) return TINV_ERR_BAD_ARG;
  if (exec_tasks) *exec_tasks = p->nexec;
  if (items) *items = p->items;
  if (edges) *edges = p->nedges;
  return TINV_OK;
}

// streamed host I/O of one tinv_plan_exec_host call
struct HostIO {
  const double* a;
  int64_t lda;
  double* xhost;  // page-locked host output
  int64_t ldx;
  int mode;
};
// device -> host copy streams of a streamed run. Few: CUDA multiplexes streams
// onto a limited set of hardware connections (CUDA_DEVICE_MAX_CONNECTIONS,
// default 8), and a stream blocked in cuStreamWaitValue32 must not share one
// with the arrival copies or the executor (TINV_DEPART_STREAMS overrides, <= 8)
constexpr int kMaxDepartStreams = 8;
static int depart_streams() {
  const char* e = getenv("TINV_DEPART_STREAMS");
  const int v = e ? atoi(e) : 4;
  return v < 1 ? 1 : (v > kMaxDepartStreams ? kMaxDepartStreams : v);
}

typedef CUresult (*PFN_batchMemOp)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);

// Copy engines: A's lower tiles into their slots in inbox order, each followed
// by its arrival flag (a stream write-value, ordered after the copy). Runs of
// tiles contiguous on both sides (batched t = 1 stores) move as one copy.
// Arrival copy runs (inbox order): runs of tiles contiguous on both sides
// (batched t = 1 stores) move as one copy. Each run is gated by ONE flag
// (gate_flag[run]): a flag write per tile costs the copy engine about half of
// its H2D rate (measured, tools/copy_probe.py).
static void tri_decode_h(int64_t k, int64_t& i, int64_t& j) {
  i = (int64_t)((std::sqrt(8.0 * (double)k + 1.0) - 1.0) * 0.5);
  while (i * (i + 1) / 2 > k) --i;
  while ((i + 1) * (i + 2) / 2 <= k) ++i;
  j = k - i * (i + 1) / 2;
}

// Column-panel runs: with unpadded tiles (b == bp) a streamed run first
// resets every tile's home slot to column-major order (its input is fully
// overwritten by the arrivals), so the tiles (i, j), (i+1, j), ... of a
// column sit in consecutive slots and one 2D copy moves up to kRunBytes of a
// column panel: ~300 copy calls at C3 instead of 2080, all enqueued before
// the executor launches.
constexpr size_t kRunBytes = 16u << 20;
static void arrival_runs(tinv_ctx* c, tinv_plan* p, const HostIO& io, std::vector<int32_t>& run_first,
                         std::vector<int32_t>& gate) {
  const int64_t na = (int64_t)p->arrive_tile.size(), n = c->n, T1 = c->T1;
  const int64_t max_run = std::max<int64_t>(1, std::min<int64_t>(128, kRunBytes / ((size_t)c->slot_elems * 8)));
  run_first.clear();
  gate.assign(std::max<int64_t>(na, 1), 0);
  for (int64_t s0 = 0; s0 < na;) {
    const int32_t o = p->arrive_tile[s0];
    int64_t run = 1;
    if (T1 == 1 && c->b == c->bp && io.lda == n) {  // batched t = 1: whole matrices, contiguous on both sides
      while (s0 + run < na && run < 64 && p->arrive_tile[s0 + run] == o + run &&
             c->a_slot[o + run] == c->a_slot[o] + run)
        ++run;
    } else if (c->b == c->bp) {  // the next tiles down the same column, in consecutive slots
      int64_t i, j;
      tri_decode_h(o % T1, i, j);
      const int64_t m0 = o / T1;
      while (s0 + run < na && run < max_run && i + run < c->t) {
        const int64_t nx = m0 * T1 + tri_index(i + run, j);
        if (p->arrive_tile[s0 + run] != nx || c->a_slot[nx] != c->a_slot[o] + run) break;
        ++run;
      }
    }
    for (int64_t r = 0; r < run; ++r) gate[s0 + r] = (int32_t)run_first.size();
    run_first.push_back((int32_t)s0);
    s0 += run;
  }
  run_first.push_back((int32_t)na);
}

static int enqueue_arrivals(tinv_ctx* c, tinv_plan* p, const HostIO& io, const std::vector<int32_t>& run_first,
                            int32_t* gate_flag, cudaStream_t st) {
  static PFN_batchMemOp batch_mem_op = nullptr;
  if (!batch_mem_op) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(c, cudaGetDriverEntryPoint("cuStreamBatchMemOp", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(c, TINV_ERR_CUDA, "cuStreamBatchMemOp unavailable");
    batch_mem_op = (PFN_batchMemOp)fn;
  }
  const int64_t b = c->b, bp = c->bp, n = c->n, T1 = c->T1;
  const size_t tile_bytes = (size_t)c->slot_elems * 8;
  for (size_t g = 0; g + 1 < run_first.size(); ++g) {
    const int64_t s0 = run_first[g], run = run_first[g + 1] - s0;
    const int32_t o = p->arrive_tile[s0];
    const int64_t m = o / T1;
    int64_t i, j;
    tri_decode_h(o % T1, i, j);
    double* dst = c->pool + (int64_t)c->a_slot[o] * c->slot_elems;
    const double* src = io.a + m * n * io.lda + i * b * io.lda + j * b;
    if (run > 1 && T1 == 1)  // whole consecutive matrices
      CK(c, cudaMemcpyAsync(dst, src, tile_bytes * run, cudaMemcpyHostToDevice, st));
    else  // one tile, or a column panel of `run` tiles into consecutive slots (b == bp)
      CK(c, cudaMemcpy2DAsync(dst, bp * 8, src, io.lda * 8, b * 8, b * run, cudaMemcpyHostToDevice, st));
    CUstreamBatchMemOpParams op{};
    op.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
    op.writeValue.address = (CUdeviceptr)(gate_flag + g);
    op.writeValue.value = 1;
    op.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
    const CUresult r = batch_mem_op((CUstream)st, 1u, &op, 0);
    if (r != CUDA_SUCCESS) return fail(c, TINV_ERR_CUDA, "arrival flag write failed (CUresult " + std::to_string(r) + ")");
  }
  return TINV_OK;
}

typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

// Copy engines, device -> host: for each copy group (departure order, spread
// over depart_streams() streams) wait until all its tiles departed, then move
// them: LOWER: the tile's final slot (renaming parity decides cur or alt) to
// block (i, j); SYMMETRIZE: off-diagonal tiles also their staged transpose to
// block (j, i), diagonal tiles their staged mirrored form.
static int enqueue_departures(tinv_ctx* c, tinv_plan* p, const HostIO& io, const std::vector<int32_t>& gfirst,
                              const std::vector<int32_t>& gsize, int64_t stage_base, cudaEvent_t after) {
  static PFN_waitValue32 wait_value = nullptr;
  if (!wait_value) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(c, cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(c, TINV_ERR_CUDA, "cuStreamWaitValue32 unavailable");
    wait_value = (PFN_waitValue32)fn;
  }
  const int nds = depart_streams();
  for (int k = 0; k < nds; ++k) {
    if (!c->dst[k]) CK(c, cudaStreamCreateWithFlags(&c->dst[k], cudaStreamNonBlocking));
    CK(c, cudaStreamWaitEvent(c->dst[k], after, 0));
  }
  const int64_t b = c->b, bp = c->bp, n = c->n, T1 = c->T1, ldx = io.ldx;
  const bool sym = io.mode == TINV_DENSE_SYMMETRIZE;
  double* X = io.xhost;
  for (size_t g = 0; g < gfirst.size(); ++g) {
    cudaStream_t s = c->dst[g % nds];
    if (wait_value((CUstream)s, (CUdeviceptr)(p->d_depart_count + g), (cuuint32_t)gsize[g], CU_STREAM_WAIT_VALUE_GEQ) !=
        CUDA_SUCCESS)
      return fail(c, TINV_ERR_CUDA, "departure wait failed");
    const int64_t k = gfirst[g], m = k / T1, kk = k % T1;
    int64_t i = (int64_t)((std::sqrt(8.0 * (double)kk + 1.0) - 1.0) * 0.5);
    while (i * (i + 1) / 2 > kk) --i;
    while ((i + 1) * (i + 2) / 2 <= kk) ++i;
    const int64_t j = kk - i * (i + 1) / 2;
    double* xm = X + m * n * ldx;
    const double* fin = c->pool + (int64_t)(p->rename_parity[k] ? alt_slot_of(c, k) : c->a_slot[k]) *
                                      c->slot_elems;
    const double* stg = c->pool + (stage_base + k) * c->slot_elems;
    if (gsize[g] > 1) {  // contiguous staged diagonal tiles of consecutive matrices
      CK(c, cudaMemcpyAsync(xm, stg, (size_t)gsize[g] * c->slot_elems * 8, cudaMemcpyDeviceToHost, s));
      continue;
    }
    if (!sym || i != j)
      CK(c, cudaMemcpy2DAsync(xm + i * b * ldx + j * b, ldx * 8, fin, bp * 8, b * 8, b, cudaMemcpyDeviceToHost, s));
    if (sym)
      CK(c, cudaMemcpy2DAsync(xm + j * b * ldx + i * b, ldx * 8, stg, bp * 8, b * 8, b, cudaMemcpyDeviceToHost, s));
  }
  return TINV_OK;
}

static int plan_exec_impl(tinv_plan* p, tinv_err* err, double* ms, const HostIO* io);

int tinv_plan_exec(tinv_plan* p, tinv_err* err, double* ms) {
  set_err(err, -1, -1, TINV_OK, -1);
  if (!p) return TINV_ERR_BAD_ARG;
  if (p->flags & TINV_STREAM_IO) return fail(p->ctx, TINV_ERR_BAD_ARG, "a TINV_STREAM_IO plan runs with tinv_plan_exec_host");
  return plan_exec_impl(p, err, ms, nullptr);
}

int tinv_plan_exec_host(tinv_plan* p, const double* a, int64_t lda, double* x, int64_t ldx, int mode, tinv_err* err,
                        double* ms) {
  set_err(err, -1, -1, TINV_OK, -1);
  if (!p) return TINV_ERR_BAD_ARG;
  tinv_ctx* c = p->ctx;
  if (!(p->flags & TINV_STREAM_IO)) return fail(c, TINV_ERR_BAD_ARG, "plan was not made with TINV_STREAM_IO");
  if (!a || !x || lda < c->n || ldx < c->n || (mode != TINV_DENSE_LOWER_TILES && mode != TINV_DENSE_SYMMETRIZE))
    return fail(c, TINV_ERR_BAD_ARG, "bad exec_host arguments");
  CK(c, cudaSetDevice(c->device));
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, x) != cudaSuccess || at.type != cudaMemoryTypeHost) {
    cudaGetLastError();
    return fail(c, TINV_ERR_BAD_ARG, "output must be page-locked host memory");
  }
  HostIO io{a, lda, x, ldx, mode};
  return plan_exec_impl(p, err, ms, &io);
}

static int plan_exec_impl(tinv_plan* p, tinv_err* err, double* ms, const HostIO* io) {
  tinv_ctx* c = p->ctx;
  const int64_t T = c->T, nx = p->nexec;
  CK(c, cudaSetDevice(c->device));
  const int64_t scratch_base = c->mslots + p->dyn_slots;
  const bool keep = (p->flags & TINV_KEEP_ON_FAILURE) != 0;
  const int64_t backup_base = scratch_base + c->nsm;
  const bool staged_out = io && io->mode == TINV_DENSE_SYMMETRIZE;
  int rc = ensure_pool(c, backup_base + ((keep || staged_out) ? T : 0));
  if (rc) return rc;
  if (nx == 0) {
    if (ms) *ms = 0.0;
    return TINV_OK;
  }
  cudaStream_t st = c->st;
  if (io && c->b == c->bp && c->T1 > 1) {
    // streamed run: the input is fully overwritten by the arrivals, so the
    // tiles get column-major home slots (column panels move as one copy)
    for (int64_t m = 0; m < c->nmat; ++m) {
      int32_t s = (int32_t)(m * c->T1);
      for (int64_t j = 0; j < c->t; ++j)
        for (int64_t i = j; i < c->t; ++i) {
          const int64_t k = m * c->T1 + tri_index(i, j);
          c->a_slot[k] = c->home[k] = s++;
        }
    }
  }
  // reset the mutable executor state
  for (int64_t k = 0; k < T; ++k) {
    p->cur0[k] = c->a_slot[k];
    p->alt0[k] = alt_slot_of(c, k);
  }
  CK(c, cudaMemcpyAsync(p->d_indeg, p->indeg0.data(), nx * 4, cudaMemcpyHostToDevice, st));
  CK(c, cudaMemsetAsync(p->d_done, 0, nx * 4, st));
  CK(c, cudaMemcpyAsync(p->d_cur, p->cur0.data(), p->nlogical * 4, cudaMemcpyHostToDevice, st));
  CK(c, cudaMemcpyAsync(p->d_alt, p->alt0.data(), p->nlogical * 4, cudaMemcpyHostToDevice, st));
  const int NQ = p->nranks * NLEV;
  CK(c, cudaMemcpyAsync(p->d_queue, p->q_init.data(), p->q_off[NQ] * 8, cudaMemcpyHostToDevice, st));
  CK(c, cudaMemsetAsync(p->d_head, 0, NQ * 4, st));
  CK(c, cudaMemcpyAsync(p->d_tail, p->tail0.data(), NQ * 4, cudaMemcpyHostToDevice, st));
  CK(c, cudaMemsetAsync(p->d_idle, 0, (size_t)c->nsm * 8, st));
  const int32_t ctr[2] = {(int32_t)nx, 0};
  CK(c, cudaMemcpyAsync(p->d_ctr, ctr, 8, cudaMemcpyHostToDevice, st));
  CK(c, cudaMemsetAsync(p->d_err, 0xff, 8, st));
  CK(c, cudaMemsetAsync(p->d_progress, 0, 4, st));
  if (p->d_ts) {
    CK(c, cudaMemsetAsync(p->d_ts, 0xff, nx * 8, st));
    CK(c, cudaMemsetAsync(p->d_te, 0, nx * 8, st));
    CK(c, cudaMemsetAsync(p->d_tsm, 0xff, nx * 4, st));
    CK(c, cudaMemsetAsync(p->d_tr, 0, nx * 8, st));
    CK(c, cudaMemsetAsync(p->d_tr + nx, 0xff, nx * 8, st));  // first claim of each task (atomicMin)
  }
  std::vector<int32_t> from(T), to(T);
  if (keep) {
    for (int64_t k = 0; k < T; ++k) {
      from[k] = c->a_slot[k];
      to[k] = (int32_t)(backup_base + k);
    }
    CK(c, cudaMemcpyAsync(p->d_snap_from, from.data(), T * 4, cudaMemcpyHostToDevice, st));
    CK(c, cudaMemcpyAsync(p->d_snap_to, to.data(), T * 4, cudaMemcpyHostToDevice, st));
    CK(c, launch_copy_slots(c->pool, c->slot_elems, p->d_snap_from, p->d_snap_to, T, st));
  }
  ExecParams P;
  memset(&P, 0, sizeof(P));
  P.pool = c->pool;
  P.slot_elems = c->slot_elems;
  P.bp = (int32_t)c->bp;
  P.R = (int32_t)c->R;
  // TINV_NO_KTRIM=1 (A/B switch): treat the padding as data, as before round 2
  static const bool no_ktrim = getenv("TINV_NO_KTRIM") && atoi(getenv("TINV_NO_KTRIM"));
  P.b = no_ktrim ? (int32_t)c->bp : (int32_t)c->b;
  P.ntasks = (int32_t)nx;
  P.scratch_base = (int32_t)scratch_base;
  P.tasks = p->d_tasks;
  P.succ = p->d_succ;
  P.indeg = p->d_indeg;
  P.done = p->d_done;
  P.cur_slot = p->d_cur;
  P.alt_slot = p->d_alt;
  P.queue = p->d_queue;
  for (int l = 0; l <= NLEV; ++l) P.q_off[l] = p->nranks == 1 ? p->q_off[l] : 0;
  P.nranks = p->nranks;
  P.q_offs = p->d_qoffs;
  P.cta_idle = p->d_idle;
  // ranks in one launch: the same number of CTAs (SMs) per rank
  p->grid = p->nranks == 1 ? c->nsm : (int64_t)p->nranks * (c->nsm / p->nranks);
  P.q_head = p->d_head;
  P.q_tail = p->d_tail;
  P.remaining = p->d_ctr;
  P.abort_flag = p->d_ctr + 1;
  P.err = p->d_err;
  P.progress = p->d_progress;
  P.trace_start = p->d_ts;
  P.trace_end = p->d_te;
  P.trace_sm = p->d_tsm;
  P.trace_ready = p->d_tr;
  P.t0 = 0;
  P.nrecv = (int32_t)p->nrecv;
  P.recv_base = (int32_t)c->mslots;
  for (int r = 0; r < MAX_RANKS; ++r)  // SEND targets: the receivers' receive bases (peer_attach / ipc_recv_bases)
    P.peer_recv_base[r] = c->peer_rbase[r] > 0 ? c->peer_rbase[r] : (int32_t)c->mslots;
  P.recv_task = p->d_recv_task;
  P.inbox = p->d_inbox;
  if (c->inbox) {  // multi-process: the exported inbox, zeroed by tinv_ipc_reset before the ranks' barrier
    if (c->inbox_len < p->nrecv) return fail(c, TINV_ERR_BAD_ARG, "exported inbox smaller than the plan's");
    P.inbox = c->inbox;
  } else {
    CK(c, cudaMemsetAsync(p->d_inbox, 0, p->recv_task_h.size() * 4, st));
  }
  for (int r = 0; r < MAX_RANKS; ++r) {  // peers: IPC-mapped pools of the other ranks, or this pool (loopback)
    P.peer_pool[r] = c->peer_pool[r] ? c->peer_pool[r] : c->pool;
    P.peer_inbox[r] = c->peer_inbox[r] ? c->peer_inbox[r] : P.inbox;
  }
  std::vector<int32_t> grp_first, grp_size;  // copy groups of departing tiles (in departure order)
  std::vector<int32_t> run_first, gate;       // arrival copy runs and entry -> run
  if (io) {
    arrival_runs(c, p, *io, run_first, gate);
    CK(c, cudaMemcpyAsync(p->d_recv_gate, gate.data(), gate.size() * 4, cudaMemcpyHostToDevice, st));
    CK(c, cudaMemsetAsync(p->d_gate_flag, 0, gate.size() * 4, st));
    P.recv_gate = p->d_recv_gate;
    P.gate_flag = p->d_gate_flag;
    P.depart_mode = io->mode;
    P.stage_base = (int32_t)backup_base;  // staging tiles (SYMMETRIZE) use the snapshot region
    // groups: runs of consecutive staged diagonal tiles that are contiguous in
    // the host matrix too (batched t = 1 stores) move as one copy
    std::vector<int32_t> hg(T, 0);
    const bool runs = io->mode == TINV_DENSE_SYMMETRIZE && c->T1 == 1 && c->b == c->bp && io->ldx == c->n;
    for (size_t x = 0; x < p->depart_tile.size(); ++x) {
      const int32_t k = p->depart_tile[x];
      if (runs && !grp_first.empty() && grp_size.back() < 64 && k == grp_first.back() + grp_size.back()) {
        grp_size.back()++;
      } else {
        grp_first.push_back(k);
        grp_size.push_back(1);
      }
      hg[k] = (int32_t)grp_first.size() - 1;
    }
    CK(c, cudaMemcpyAsync(p->d_depart_group, hg.data(), T * 4, cudaMemcpyHostToDevice, st));
    CK(c, cudaMemsetAsync(p->d_depart_count, 0, T * 4, st));
    CK(c, cudaMemsetAsync(p->d_depart_seq + T, 0, 4, st));
    P.depart_group = p->d_depart_group;
    P.depart_count = p->d_depart_count;
    P.depart_seq = p->d_depart_seq;
    P.depart_seq_ctr = p->d_depart_seq + T;
    if (c->bp != c->b) {  // padding of the arriving tiles (the copies move the b x b part only)
      CK(c, cudaMemcpyAsync(c->d_a_slot, c->a_slot.data(), c->T * sizeof(int32_t), cudaMemcpyHostToDevice, st));
      CK(c, launch_pad(c->pool, c->slot_elems, c->d_a_slot, (int)c->b, (int)c->bp, c->T, c->T1, st));
    }
  }
  {
    const char* pf = getenv("TINV_PREFETCH_MIN");
    P.prefetch_min = pf ? atoi(pf) : kPrefetchMin;
    const char* tk = getenv("TINV_TICKET_MIN");
    P.ticket_min = tk ? std::max(1, atoi(tk)) : kTicketMin;
  }
  if (getenv("TINV_PHASE_PROFILE")) {
    if (!p->d_phase) CK(c, cudaMalloc(&p->d_phase, (size_t)c->nsm * NPHASE * 8));
    CK(c, cudaMemsetAsync(p->d_phase, 0, (size_t)c->nsm * NPHASE * 8, st));
    P.phase = p->d_phase;
  }
  CK(c, cudaEventRecord(p->ev0, st));
  if (io) {
    // Arrival copies (and their gate-flag writes) are enqueued BEFORE the
    // persistent executor, which spins on those flags: they depend only on the
    // state reset (ev0), never on the kernel, so they complete even when the
    // launch is serialised (CUDA_LAUNCH_BLOCKING, a profiler's kernel replay,
    // one hardware connection) -- forward progress by construction.
    CK(c, cudaStreamWaitEvent(c->st2, p->ev0, 0));
    const int rc2 = enqueue_arrivals(c, p, *io, run_first, p->d_gate_flag, c->st2);
    if (rc2) {
      cudaDeviceSynchronize();
      return rc2;
    }
  }
  CK(c, launch_exec(c->tmK, c->tmM, c->tmE, P, (int)c->b, (int)p->grid, st));
  CK(c, cudaEventRecord(p->ev1, st));
  if (io)  // executor done (or aborted): release every copy group still waiting
    CK(c, cudaMemsetAsync(p->d_depart_count, 0x7f, T * 4, st));
  if (io) {  // departure copies wait on counters the executor bumps; the kernel never waits on them
    const int rc2 = enqueue_departures(c, p, *io, grp_first, grp_size, backup_base, p->ev0);
    if (rc2) {
      cudaStreamSynchronize(st);
      cudaDeviceSynchronize();
      return rc2;
    }
  }
  CK(c, cudaStreamSynchronize(st));
  if (io) {
    CK(c, cudaStreamSynchronize(c->st2));
    for (int k = 0; k < kMaxDepartStreams; ++k)
      if (c->dst[k]) CK(c, cudaStreamSynchronize(c->dst[k]));
  }
  if (ms) {
    float f = 0.f;
    cudaEventElapsedTime(&f, p->ev0, p->ev1);
    *ms = f;
  }
  unsigned long long ekey = 0;
  int32_t ctr_out[2];
  CK(c, cudaMemcpy(&ekey, p->d_err, 8, cudaMemcpyDeviceToHost));
  CK(c, cudaMemcpy(ctr_out, p->d_ctr, 8, cudaMemcpyDeviceToHost));
  if (p->d_ts) {
    p->h_ts.resize(nx);
    p->h_te.resize(nx);
    p->h_tsm.resize(nx);
    CK(c, cudaMemcpy(p->h_ts.data(), p->d_ts, nx * 8, cudaMemcpyDeviceToHost));
    CK(c, cudaMemcpy(p->h_te.data(), p->d_te, nx * 8, cudaMemcpyDeviceToHost));
    CK(c, cudaMemcpy(p->h_tsm.data(), p->d_tsm, nx * 4, cudaMemcpyDeviceToHost));
    if (getenv("TINV_READY_PROFILE")) {  // dispatch delay: ready (in-degree 0) -> first item start
      std::vector<unsigned long long> tr(2 * nx);
      CK(c, cudaMemcpy(tr.data(), p->d_tr, 2 * nx * 8, cudaMemcpyDeviceToHost));
      static const char* kn[] = {"COPY", "POTRF", "TRSM", "SYRK_SUB", "SYRK_ADD_T", "GEMM", "TRTRI", "TRMM_L",
                                 "TRMM_RN", "TRMM_LT", "LAUUM", "INV", "SEND", "RECV", "ARRIVE", "DEPART", "POTRF_INV"};
      double sum[17] = {0}, mx[17] = {0};
      int cnt[17] = {0};
      for (int64_t u = 0; u < nx; ++u) {
        const int k = p->tasks[u].kind;
        if (k < 0 || k > 16 || p->h_ts[u] == ~0ull) continue;
        const double d = tr[u] ? ((double)p->h_ts[u] - (double)tr[u]) * 1e-3 : 0.0;  // us
        sum[k] += d;
        mx[k] = std::max(mx[k], d);
        ++cnt[k];
      }
      fprintf(stderr, "[tinv ready] dispatch delay per kind (tasks, mean us, max us):");
      for (int k = 0; k < 17; ++k)
        if (cnt[k]) fprintf(stderr, " %s %d %.1f %.1f |", kn[k], cnt[k], sum[k] / cnt[k], mx[k]);
      fprintf(stderr, "\n");
      // split: ready -> first claim by a producer (queueing) and claim -> first item start (the
      // claiming CTA's consumers still busy / operands streaming)
      double q[17] = {0}, w[17] = {0}, qm[17] = {0}, wm[17] = {0};
      for (int64_t u = 0; u < nx; ++u) {
        const int k = p->tasks[u].kind;
        if (k < 0 || k > 16 || p->h_ts[u] == ~0ull || !tr[u] || tr[nx + u] == ~0ull) continue;
        const double a = ((double)tr[nx + u] - (double)tr[u]) * 1e-3, b = ((double)p->h_ts[u] - (double)tr[nx + u]) * 1e-3;
        q[k] += a, w[k] += b, qm[k] = std::max(qm[k], a), wm[k] = std::max(wm[k], b);
      }
      fprintf(stderr, "[tinv ready] ready->claim / claim->start per kind (mean us, max us):");
      for (int k = 0; k < 17; ++k)
        if (cnt[k]) fprintf(stderr, " %s %.1f/%.1f %.1f/%.1f |", kn[k], q[k] / cnt[k], qm[k], w[k] / cnt[k], wm[k]);
      fprintf(stderr, "\n");
    }
  }
  if (p->d_ts && io && getenv("TINV_DEPART_PROFILE")) {  // when do result tiles become final?
    unsigned long long t0 = ~0ull, t1 = 0;
    std::vector<unsigned long long> de, ar;
    for (int64_t u = 0; u < nx; ++u) {
      if (p->h_ts[u] != ~0ull) t0 = std::min(t0, p->h_ts[u]);
      t1 = std::max(t1, p->h_te[u]);
      if (p->tasks[u].kind == KIND_DEPART) de.push_back(p->h_te[u]);
      if (p->tasks[u].kind == KIND_ARRIVE) ar.push_back(p->h_te[u]);
    }
    for (auto* v : {&ar, &de}) {
      std::sort(v->begin(), v->end());
      fprintf(stderr, "[tinv %s] run %.1f ms; tiles at (ms): ", v == &ar ? "arrive" : "depart", (t1 - t0) * 1e-6);
      for (double q : {0.1, 0.25, 0.5, 0.75, 0.9, 0.99, 1.0})
        fprintf(stderr, "q%.2f %.1f ", q, ((*v)[std::min(v->size() - 1, (size_t)(q * v->size()))] - t0) * 1e-6);
      fprintf(stderr, "\n");
    }
  }
  if (p->d_phase) {
    std::vector<unsigned long long> ph((size_t)c->nsm * NPHASE);
    CK(c, cudaMemcpy(ph.data(), p->d_phase, ph.size() * 8, cudaMemcpyDeviceToHost));
    double tot[NPHASE] = {0};
    for (int x = 0; x < c->nsm; ++x)
      for (int k = 0; k < NPHASE; ++k) tot[k] += (double)ph[x * NPHASE + k];
    const double items = tot[6] > 0 ? tot[6] : 1;
    fprintf(stderr,
            "[tinv phase] per item (cycles): item-wait %.0f mainloop %.0f epilogue %.0f job-end %.0f item-end %.0f "
            "completion %.0f | items %.0f jobs %.0f | special totals: load %.0f factor %.0f inverse %.0f store %.0f\n",
            tot[0] / items, tot[1] / items, tot[2] / items, tot[3] / items, tot[4] / items, tot[5] / items, tot[6],
            tot[7], tot[8], tot[9], tot[10], tot[11]);
    fprintf(stderr, "[tinv phase] trtri base %.0f l16 %.0f l32 %.0f l64 %.0f\n", tot[15], tot[16], tot[17], tot[18]);
    const double pops = tot[23] > 0 ? tot[23] : 1;
    fprintf(stderr,
            "[tinv phase] producer per pop: slot-wait %.0f pop %.0f produce %.0f (pops %.0f) | storer per item: "
            "quarters %.0f job-end %.0f item-end %.0f idle %.0f\n",
            tot[20] / pops, tot[21] / pops, tot[22] / pops, tot[23], tot[24] / items, tot[25] / items,
            tot[26] / items, tot[27] / items);
    fprintf(stderr, "[tinv phase] consumer idle (item-wait) share of the SMs per ~1 ms bin:");
    for (int k = 0; k < PHASE_NBIN; ++k)
      if (tot[PHASE_BIN0 + k] > 0) fprintf(stderr, " %d:%.3f", k, tot[PHASE_BIN0 + k] / (c->nsm * 1048576.0 * 1.965));
    fprintf(stderr, "\n");
  }
  if (ekey != ~0ull || ctr_out[0] != 0) {
    if (keep) {
      CK(c, cudaMemcpyAsync(p->d_snap_from, to.data(), T * 4, cudaMemcpyHostToDevice, st));
      CK(c, cudaMemcpyAsync(p->d_snap_to, from.data(), T * 4, cudaMemcpyHostToDevice, st));
      CK(c, launch_copy_slots(c->pool, c->slot_elems, p->d_snap_from, p->d_snap_to, T, st));
      CK(c, cudaStreamSynchronize(st));
    }
    if (ekey == ~0ull) {
      set_err(err, -1, -1, TINV_ERR_INTERNAL, -1);
      return fail(c, TINV_ERR_INTERNAL, "executor finished with " + std::to_string(ctr_out[0]) + " tasks pending");
    }
    const int32_t task = (int32_t)(ekey >> 32);
    const int32_t code = (int32_t)((ekey >> 24) & 0xff);
    const int32_t index = (int32_t)(ekey & 0xffffff);
    if (code == TINV_ERR_INTERNAL) {
      set_err(err, -1, -1, code, -1);
      return fail(c, code, "executor watchdog: no progress");
    }
    set_err(err, task, task >= 0 && task < p->nref ? p->ref_kind[task] : -1, code, index);
    return fail(c, code, "task " + std::to_string(task) + " failed");
  }
  // success: adopt the renamed slots of the matrix tiles
  CK(c, cudaMemcpy(c->a_slot.data(), p->d_cur, T * 4, cudaMemcpyDeviceToHost));
  p->h_idle.resize(p->grid);
  CK(c, cudaMemcpy(p->h_idle.data(), p->d_idle, p->grid * 8, cudaMemcpyDeviceToHost));
  if (io && !(c->T1 == 1 && c->b == c->bp)) {  // next run: enqueue departures in the observed order
    std::vector<int32_t> seq(T);
    CK(c, cudaMemcpy(seq.data(), p->d_depart_seq, T * 4, cudaMemcpyDeviceToHost));
    p->depart_tile.swap(seq);
  }
  return TINV_OK;
}

int tinv_plan_trace(const tinv_plan* p, int64_t* start_ns, int64_t* end_ns, int32_t* sm, int64_t ntasks) {
  if (!p || ntasks < p->nref || p->h_ts.empty()) return TINV_ERR_BAD_ARG;
  unsigned long long base = ~0ull;
  for (int64_t u = 0; u < p->nexec; ++u)
    if (p->exec_ref[u] >= 0) base = std::min(base, p->h_ts[u]);
  for (int64_t r = 0; r < p->nref; ++r) {
    start_ns[r] = -1;
    end_ns[r] = -1;
    sm[r] = -1;
  }
  for (int64_t u = 0; u < p->nexec; ++u) {
    const int32_t r = p->exec_ref[u];
    if (r < 0) continue;  // ARRIVE / DEPART
    const int64_t s = (int64_t)(p->h_ts[u] - base), e = (int64_t)(p->h_te[u] - base);
    if (start_ns[r] < 0 || s < start_ns[r]) start_ns[r] = s;
    if (e > end_ns[r]) {
      end_ns[r] = e;
      sm[r] = p->h_tsm[u];
    }
  }
  return TINV_OK;
}

int tinv_run(tinv_ctx* c, const int32_t* table, int64_t n, int32_t stream_t, const int64_t* barriers, int64_t nbar,
             uint32_t flags, tinv_err* err) {
  tinv_plan* p = nullptr;
  int rc = tinv_plan_create(c, table, n, stream_t, barriers, nbar, flags, &p, err);
  if (rc) return rc;
  rc = tinv_plan_exec(p, err, nullptr);
  tinv_plan_destroy(p);
  return rc;
}

}  // extern "C"
