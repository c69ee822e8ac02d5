// tsa_api.cu -- host side of libtsa: argument validation, workspace carving and
// launch sequencing behind the C ABI declared in include/tsa.h.  Never
// allocates device memory, never synchronises the caller's stream (except the
// documented blocking tsa_segment_host), keeps no global mutable state other
// than the thread-local error string.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "tsa.h"
#include "tsa_internal.h"
#include "tsa_kernels.cuh"
#include "k_fused.cuh"
#include "k_stream.cuh"

namespace {

thread_local std::string g_last_error;

int g_num_sms();

tsa_status set_error(tsa_status s, const char *msg) {
  g_last_error = msg;
  return s;
}

tsa_status check_cuda(const char *where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[512];
    snprintf(buf, sizeof(buf), "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
    return set_error(TSA_ERR_CUDA, buf);
  }
  return TSA_OK;
}

#define TSA_CUDA(call)                                                        \
  do {                                                                        \
    cudaError_t _e = (call);                                                  \
    if (_e != cudaSuccess) {                                                  \
      char _b[512];                                                           \
      snprintf(_b, sizeof(_b), "%s: %s", #call, cudaGetErrorString(_e));      \
      return set_error(TSA_ERR_CUDA, _b);                                     \
    }                                                                         \
  } while (0)

#define TSA_TRY(expr)               \
  do {                              \
    tsa_status _s = (expr);         \
    if (_s != TSA_OK) return _s;    \
  } while (0)

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// bump allocator over a caller-provided workspace (sizes only when base == null)
struct Carve {
  char *base;
  size_t off = 0;
  template <typename T>
  T *take(size_t count) {
    T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
    off += align_up(count * sizeof(T));
    return p;
  }
};

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

double binom_d(double n, int r) {
  double v = 1.0;
  for (int i = 0; i < r; i++) v = v * (n - i) / (i + 1);
  return v;
}

bool valid_search_shape(int64_t nz, int64_t N, int32_t bins, int32_t k, double q,
                        int32_t objective, int32_t enumeration) {
  if (nz <= 0 || nz > 65535 || N <= 0 || N >= (int64_t(1) << 31)) return false;
  if (bins < 2 || bins > TSA_BINS_MAX) return false;
  if (k < 1 || k > TSA_KMAX || k > bins - 1) return false;
  if (!(q > 0.0) || !std::isfinite(q)) return false;
  if (objective != TSA_OBJ_PSEUDO_ADDITIVE && objective != TSA_OBJ_SUM_PLUS_PRODUCT) return false;
  if (enumeration != TSA_ENUM_CANONICAL && enumeration != TSA_ENUM_FULL && enumeration != TSA_ENUM_DP)
    return false;
  if (enumeration == TSA_ENUM_DP && objective != TSA_OBJ_PSEUDO_ADDITIVE) return false;
  if (binom_d((double)bins - 1, k) >= 9.2e18) return false;
  return true;
}

int search_mode(double q, int32_t objective) {
  if (objective == TSA_OBJ_SUM_PLUS_PRODUCT) return tsa::SPP;
  if (q == 1.0) return tsa::SUM;
  return q < 1.0 ? tsa::PROD_MAX : tsa::PROD_MIN;
}

// Luts for q: the small table pointer plus the Horner coefficients
// (binom(-q, k) and log1p(d)/d), computed here once per call in fp64.
tsa::Luts make_luts(double q, const double *sp) {
  tsa::Luts l = {};
  const bool shannon = q == 1.0;
  l.sp = sp;
  l.c[0] = 1.0;
  for (int k = 1; k <= 12; k++) l.c[k] = l.c[k - 1] * (-q - (k - 1)) / k;
  for (int k = 0; k <= 6; k++) l.lc[k] = (k & 1 ? -1.0 : 1.0) / (k + 1);
  // truncation |binom(-q, deg+1)| d^(deg+1), d < 2^-10: deg 5 is < 2^-57 for q <= 2
  l.deg = q <= 2.0 ? 5 : q <= 10.0 ? 6 : 12;
  for (int s = 0; s < 32; s++) {
    const double x = std::ldexp(1.0, s);
    l.p2[s] = shannon ? std::log(x) : 1.0 / std::pow(x, q);
  }
  l.iqm1 = shannon ? 0.0 : 1.0 / (q - 1.0);
  l.omq = 1.0 - q;
  l.shannon = shannon;
  return l;
}

// R-table row stride: >= bins + 8 (8-column groups read past M-2 into NaN) and even
inline int rstride(int32_t bins) { return (bins + 8 + 1) & ~1; }

bool use_rtable(int32_t bins, int32_t k, int32_t objective) {
  return objective == TSA_OBJ_PSEUDO_ADDITIVE && k >= 3 && bins <= 512;
}

struct SearchWs {
  double *sp = nullptr;  // small class-term table (Luts::sp)
  uint32_t *cC = nullptr, *fC = nullptr;
  double *cWhi = nullptr, *cWlo = nullptr, *fWhi = nullptr, *fWlo = nullptr;
  int32_t *cBin = nullptr, *fBin = nullptr;
  double *Asuf = nullptr, *R = nullptr, *PP = nullptr, *AI = nullptr;
  int32_t *M = nullptr;
  int32_t *counter = nullptr;  // dynamic work-item counter of the k >= 3 / k = 2 search
  int32_t *mmax = nullptr;     // max M over slices (k = 2 block search)
  double *item_score = nullptr;  // [nb][nz] k = 2 a-block partials
  uint64_t *item_key = nullptr;
  tsa::K2Row *rows = nullptr;    // [nz][k2_row_stride] packed positions (k = 2)
  int32_t *ccur = nullptr;       // [nz] per-slice chunk counters (k_search_tri)
  double *seed = nullptr;        // [nz] seed scores of the pruned k = 2 search
  tsa::K2Chk *chk = nullptr;     // [2][nz][k2_row_stride] bound records of the pruned k = 2 search
};

constexpr int kTriSS = 8;  // k_search_tri: CTA entries per slice

// row stride of the k = 2 packed positions: entries 0..bins plus the rows the
// kernel reads past a slice's end (kK2Rows)
inline int k2_row_stride(int32_t bins) { return bins + 1 + 8; }

// a-blocks of 32 first thresholds of the k = 2 block search (upper bound: M <= bins)
inline int k2_blocks(int32_t bins) { return bins >= 3 ? (bins - 3) / 32 + 1 : 1; }

size_t carve_search(Carve &c, SearchWs &w, int64_t nz, int64_t N, int32_t bins, int32_t k,
                    double q, int32_t objective, int32_t enumeration) {
  const size_t E = (size_t)bins + 1;
  (void)N;
  (void)q;
  w.sp = c.take<double>(tsa::kSmallLut);
  // + kPad entries: the k = 2 kernel reads up to kK2Rows rows past a slice's end
  const size_t kPad = 8;
  w.cC = c.take<uint32_t>(nz * E + kPad);
  w.cWhi = c.take<double>(nz * E + kPad);
  w.cWlo = c.take<double>(nz * E + kPad);
  w.cBin = c.take<int32_t>(nz * E + kPad);
  if (enumeration == TSA_ENUM_FULL) {
    w.fC = c.take<uint32_t>(nz * E + kPad);
    w.fWhi = c.take<double>(nz * E + kPad);
    w.fWlo = c.take<double>(nz * E + kPad);
    w.fBin = c.take<int32_t>(nz * E + kPad);
  }
  w.Asuf = c.take<double>(nz * (size_t)bins + kPad);
  w.M = c.take<int32_t>(nz);
  w.counter = c.take<int32_t>(2);
  w.mmax = w.counter + 1;
  if (k >= 3) {  // k_search_tri: entry slots [kTriSS][nz] and per-slice chunk counters
    w.item_score = c.take<double>((size_t)kTriSS * nz);
    w.item_key = c.take<uint64_t>((size_t)kTriSS * nz);
    w.ccur = c.take<int32_t>(nz);
  }
  if (k == 2) {
    w.item_score = c.take<double>((size_t)k2_blocks(bins) * tsa::k2_tiles(bins) * nz);
    w.item_key = c.take<uint64_t>((size_t)k2_blocks(bins) * tsa::k2_tiles(bins) * nz);
    w.rows = c.take<tsa::K2Row>(nz * (size_t)k2_row_stride(bins) + kPad);
    w.seed = c.take<double>(nz);
    w.chk = c.take<tsa::K2Chk>(2 * nz * (size_t)k2_row_stride(bins) + kPad);
  }
  if (use_rtable(bins, k, objective) && enumeration != TSA_ENUM_DP) {
    // (k_search_tri regions: tri_slice_stride(bins) doubles per slice)
    w.R = c.take<double>(nz * (size_t)std::max<int64_t>((int64_t)bins * rstride(bins), tsa::tri_slice_stride(bins)) + 16);
    if (enumeration == TSA_ENUM_FULL) {  // k_search_rows' prefix tables (k_search_tri needs R only)
      w.PP = c.take<double>(nz * (size_t)bins * rstride(bins) + 16);
      if (k >= 4) w.AI = c.take<double>(nz * (size_t)bins * rstride(bins) + 16);
    }
  }
  return c.off;
}

template <int K, int MODE, bool RT>
void launch_search_kr(const tsa::SearchArgs &a, dim3 grid, cudaStream_t s) {
  // stage the slice tables in shared memory when they are small
  const size_t smem = (size_t)(2 * a.E + a.L) * sizeof(double) + (size_t)a.E * sizeof(uint32_t);
  if (a.L <= 1024)
    tsa::k_search<K, MODE, RT, true><<<grid, 256, smem, s>>>(a);
  else
    tsa::k_search<K, MODE, RT, false><<<grid, 256, 0, s>>>(a);
}

template <int K, int MODE>
void launch_search_k(const tsa::SearchArgs &a, dim3 grid, cudaStream_t s, bool rt) {
  if (rt)
    launch_search_kr<K, MODE, true>(a, grid, s);
  else
    launch_search_kr<K, MODE, false>(a, grid, s);
}

template <int MODE>
void launch_search_mode(int k, const tsa::SearchArgs &a, dim3 grid, cudaStream_t s, bool rt) {
  // k >= 3 with the R table (even row stride for 16-byte pair loads): thread-per-row kernel
  if constexpr (MODE != tsa::SPP) {
    if (rt && k >= 3) {
      // persistent: 3 CTAs per SM fetch (slice, unit) items dynamically
      const int64_t items = (int64_t)grid.x * grid.y;
      cudaMemsetAsync(a.counter, 0, sizeof(int32_t), s);
      const unsigned g1 = (unsigned)std::min<int64_t>(items, 3 * g_num_sms());
      const unsigned g2 = (unsigned)std::min<int64_t>(items, 2 * g_num_sms());
      (void)g2;
      if (k == 3) {
        tsa::k_search_rows<3, MODE><<<g1, 256, 0, s>>>(a);
      } else {
        tsa::k_search_rows<4, MODE><<<g1, 256, 0, s>>>(a);
      }
      return;
    }
  }
  // k <= 2: flattened tuple-parallel kernel (tables staged in shared memory)
  if constexpr (MODE != tsa::SPP) {
    if (k <= 2) {
      const size_t smem = (size_t)(2 * a.E + 2 * a.L + tsa::kSmallLut) * sizeof(double) +
                          (size_t)a.E * sizeof(uint32_t);
      // large tables fill shared memory: one 1024-thread CTA per SM instead
      const bool big = a.L > 1024;
      auto f = big ? (k == 1 ? tsa::k_search_flat<1, MODE, 1024> : tsa::k_search_flat<2, MODE, 1024>)
                   : (k == 1 ? tsa::k_search_flat<1, MODE, 256> : tsa::k_search_flat<2, MODE, 256>);
      if (smem > 48 * 1024) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      f<<<grid, big ? 1024 : 256, smem, s>>>(a);
      return;
    }
  }
  switch (k) {
    case 1: launch_search_k<1, MODE>(a, grid, s, false); break;
    case 2: launch_search_k<2, MODE>(a, grid, s, false); break;
    case 3: launch_search_k<3, MODE>(a, grid, s, rt); break;
    default: launch_search_k<4, MODE>(a, grid, s, rt); break;
  }
}

template <int MODE>
void launch_scan(const tsa::ScanArgs &a, cudaStream_t s) {
  const size_t smem = (size_t)a.L * sizeof(double) + 1024 + (size_t)a.L * sizeof(uint32_t);
  if (smem > 48 * 1024) cudaFuncSetAttribute(tsa::k_scan<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tsa::k_scan<MODE><<<(unsigned)a.nz, tsa::kTableThreads, smem, s>>>(a);
}

template <int MODE>
void launch_rtable(const SearchWs &w, const uint32_t *C, const double *Whi, const double *Wlo,
                   const int32_t *status, int64_t nz, int E, int L, const tsa::Luts &l,
                   cudaStream_t s) {
  tsa::k_rtable<MODE><<<(unsigned)nz, 256, 0, s>>>(C, Whi, Wlo, w.Asuf, w.M, status, w.R, w.PP, w.AI, E, L,
                                            rstride(L), l);
}

int g_num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
      sms = 148;
  }
  return sms;
}

}  // namespace

extern "C" {

int32_t tsa_version(void) { return TSA_VERSION; }

const char *tsa_last_error(void) { return g_last_error.c_str(); }

void tsa_internal_set_error(const char *msg) { g_last_error = msg ? msg : ""; }

const char *tsa_status_string(tsa_status s) {
  switch (s) {
    case TSA_OK: return "TSA_OK";
    case TSA_ERR_INVALID_ARG: return "TSA_ERR_INVALID_ARG";
    case TSA_ERR_LEVEL_OVERFLOW: return "TSA_ERR_LEVEL_OVERFLOW";
    case TSA_ERR_NO_VALID_SPLIT: return "TSA_ERR_NO_VALID_SPLIT";
    case TSA_ERR_WORKSPACE: return "TSA_ERR_WORKSPACE";
    case TSA_ERR_CUDA: return "TSA_ERR_CUDA";
    case TSA_ERR_NCCL: return "TSA_ERR_NCCL";
  }
  return "TSA_ERR_UNKNOWN";
}

tsa_status tsa_validate(const tsa_problem *p) {
  if (!p) return set_error(TSA_ERR_INVALID_ARG, "problem is NULL");
  if (!p->volume) return set_error(TSA_ERR_INVALID_ARG, "volume is NULL");
  if (p->dtype != TSA_U8 && p->dtype != TSA_U16) return set_error(TSA_ERR_INVALID_ARG, "dtype");
  if (p->nx <= 0 || p->ny <= 0 || p->nz <= 0) return set_error(TSA_ERR_INVALID_ARG, "dims must be > 0");
  if (p->nz > 65535) return set_error(TSA_ERR_INVALID_ARG, "nz > 65535 (one grid row per slice)");
  if (p->nx * p->ny >= (int64_t(1) << 31)) return set_error(TSA_ERR_INVALID_ARG, "slice too large");
  if (p->dtype == TSA_U8 && p->bins > 256) return set_error(TSA_ERR_INVALID_ARG, "bins > 256 with u8");
  if (p->units_per_slice < 0 || p->units_per_slice > 65535)
    return set_error(TSA_ERR_INVALID_ARG, "units_per_slice");
  if (!valid_search_shape(p->nz, p->nx * p->ny, p->bins, p->k, p->q, p->objective, p->enumeration))
    return set_error(TSA_ERR_INVALID_ARG, "bins/k/q/objective/enumeration out of range");
  return TSA_OK;
}

int32_t tsa_default_units(int64_t nz, int32_t bins, int32_t k, int32_t enumeration) {
  return tsa_units_for_sms(nz, bins, k, enumeration, g_num_sms());
}

int32_t tsa_units_for_sms(int64_t nz, int32_t bins, int32_t k, int32_t enumeration, int32_t sms) {
  if (nz <= 0 || enumeration == TSA_ENUM_DP) return 1;
  // k <= 2: the search kernels balance their work internally (k = 2: per-warp
  // a-block items from a global queue), so one unit per slice
  if (k <= 2) return 1;
  // k_search_tri balances a slice's rows over several CTAs itself (per-slice
  // chunk counters): one unit per slice (units only partition ranks)
  if (k >= 3 && enumeration == TSA_ENUM_CANONICAL && bins <= 512) return 1;
  const double target = (double)sms * (k >= 3 ? 64.0 : 8.0);
  double rows = binom_d((double)bins - 1, k - 1);
  if (enumeration == TSA_ENUM_CANONICAL) rows = binom_d(0.45 * (bins - 1), k - 1);
  double u = std::ceil(target / (double)nz);
  // k >= 3: a unit should fill a 256-thread CTA walking 8 rows per thread
  u = std::min(u, std::max(1.0, rows / (k >= 3 ? 2048.0 : 16.0)));
  return (int32_t)std::max(1.0, std::min(u, 256.0));
}

size_t tsa_search_workspace_size(int64_t nz, int64_t N, int32_t bins, int32_t k, double q,
                                 int32_t objective, int32_t enumeration) {
  if (!valid_search_shape(nz, N, bins, k, q, objective, enumeration)) return 0;
  Carve c{nullptr};
  SearchWs w;
  return carve_search(c, w, nz, N, bins, k, q, objective, enumeration);
}

static int32_t units_of(const tsa_problem *p) {
  return p->units_per_slice > 0 ? p->units_per_slice
                                : tsa_default_units(p->nz, p->bins, p->k, p->enumeration);
}

struct SegWs {
  uint32_t *hist;
  int32_t *status;
  double *ps;
  uint64_t *pk;
  char *search;
  size_t search_bytes;
  // fused pipeline
  uint32_t *partial;
  int32_t *povf;
  int32_t *counters;
  double *luts;
  // stream pipeline: [3 + 6 nz] counters and flags, per-tile partials
  int32_t *sctr;
  double *st_score;
  uint64_t *st_key;
};

// tiles of a slice in the stream pipeline: a-blocks x second-threshold tiles
static int stream_tiles(int32_t bins) { return k2_blocks(bins) * ((bins - 2) / tsa::kStTileB + 1); }

// fused-pipeline constants (tuned on B200, profiles/)
constexpr int kFusedHC = 2;   // histogram chunks per slice (persistent fused kernel)
constexpr int kCompactHC = 4; // histogram chunks per slice (3-kernel compact path)
constexpr int kCompactLC = 4; // label chunks per slice (3-kernel compact path)
constexpr int kFusedLC = 2;   // label chunks per slice
constexpr int kFusedThreads = 512;

static bool fused_eligible(const tsa_problem *p) {
  const int64_t n = p->nx * p->ny;
  return p->k <= 2 && p->bins <= 1024 && p->enumeration == TSA_ENUM_CANONICAL &&
         p->objective == TSA_OBJ_PSEUDO_ADDITIVE && n % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(p->volume) & 15) == 0;
}

static size_t carve_segment(const tsa_problem *p, char *base, SegWs *o) {
  Carve c{base};
  const int32_t U = units_of(p);
  SegWs w;
  w.hist = c.take<uint32_t>((size_t)p->nz * p->bins);
  w.status = c.take<int32_t>((size_t)p->nz);
  w.ps = c.take<double>((size_t)U * p->nz);
  w.pk = c.take<uint64_t>((size_t)U * p->nz);
  w.search_bytes = tsa_search_workspace_size(p->nz, p->nx * p->ny, p->bins, p->k, p->q,
                                             p->objective, p->enumeration);
  w.search = c.take<char>(w.search_bytes);
  w.partial = c.take<uint32_t>((size_t)p->nz * std::max(kFusedHC, kCompactHC) * p->bins);
  w.povf = c.take<int32_t>((size_t)p->nz * std::max(kFusedHC, kCompactHC));
  w.counters = c.take<int32_t>(2 + 2 * (size_t)p->nz);
  w.luts = c.take<double>(tsa::kSmallLut);
  w.sctr = c.take<int32_t>(3 + tsa::kStCounters * (size_t)p->nz);
  const size_t nt = p->k == 2 ? (size_t)stream_tiles(p->bins) * p->nz : 0;
  w.st_score = c.take<double>(nt);
  w.st_key = c.take<uint64_t>(nt);
  if (o) *o = w;
  return c.off;
}

// stream pipeline (k_stream.cuh): k = 2, canonical, pseudo-additive, 16-voxel
// vectors; the default for bins > 1024 (the compact path covers <= 1024)
static bool stream_eligible(const tsa_problem *p) {
  const int64_t n = p->nx * p->ny;
  return p->k == 2 && p->bins >= 3 && p->enumeration == TSA_ENUM_CANONICAL &&
         p->objective == TSA_OBJ_PSEUDO_ADDITIVE && n % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(p->volume) & 15) == 0;
}
// auto-selection of the stream pipeline (kStreamAuto): off until it beats the
// staged kernels on c5 (profiles/r2*)
constexpr bool kStreamAuto = false;
static bool stream_default(const tsa_problem *p) {
  return kStreamAuto && p->pipeline == 0 && p->bins > 1024 && stream_eligible(p);
}
// the overlap pipeline (segment_overlap) by default where the search is heavy
// and not covered by compact: k = 2 above 1024 bins (c5) with enough slices
constexpr bool kOverlapAuto = false;  // enabled once measured faster (profiles/r2*)
static bool overlap_default(const tsa_problem *p) {
  return kOverlapAuto && p->pipeline == 0 && p->k == 2 && p->bins > 1024 && p->nz >= 16 &&
         p->enumeration != TSA_ENUM_DP;
}

}  // extern "C"

template <typename T, int K>
static void launch_fused_k(const tsa::FusedArgs &a, int mode, size_t smem, int grid, cudaStream_t s) {
  switch (mode) {
    case tsa::PROD_MAX: {
      auto f = tsa::k_fused<T, K, tsa::PROD_MAX>;
      if (smem > 48 * 1024) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      f<<<grid, kFusedThreads, smem, s>>>(a);
    } break;
    case tsa::PROD_MIN: {
      auto f = tsa::k_fused<T, K, tsa::PROD_MIN>;
      if (smem > 48 * 1024) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      f<<<grid, kFusedThreads, smem, s>>>(a);
    } break;
    default: {
      auto f = tsa::k_fused<T, K, tsa::SUM>;
      if (smem > 48 * 1024) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      f<<<grid, kFusedThreads, smem, s>>>(a);
    } break;
  }
}

extern "C" {

static tsa_status segment_fused(const tsa_problem *p, const tsa_outputs *out, const SegWs &w,
                                cudaStream_t s, bool persistent) {
  const int64_t N = p->nx * p->ny;
  const bool shannon = p->q == 1.0;
  tsa::FusedArgs a;
  a.vol = reinterpret_cast<const uint8_t *>(p->volume);
  a.dtype_bytes = p->dtype == TSA_U8 ? 1 : 2;
  a.n = N;
  a.nz = p->nz;
  a.L = p->bins;
  a.k = p->k;
  a.q = p->q;
  a.mode = search_mode(p->q, p->objective);
  a.thresholds = out->thresholds;
  a.objective = out->objective;
  a.hist = out->histogram ? out->histogram : w.hist;
  a.status = w.status;
  a.status2 = out->slice_status;
  a.labels = out->labels;
  a.partial = w.partial;
  a.povf = w.povf;
  a.counters = w.counters;
  a.sp = w.luts;
  a.luts = make_luts(p->q, w.luts);
  a.HC = kFusedHC;
  a.LC = kFusedLC;
  a.SB = p->slab_slices > 0 ? p->slab_slices : 16;
  a.DM = 2;
  a.DL = p->label_lag > 0 ? std::max(a.DM + 1, p->label_lag) : 6;
  a.nslab = (int)((p->nz + a.SB - 1) / a.SB);
  a.lut_per = 1024;
  a.nlut = (tsa::kSmallLut + a.lut_per - 1) / a.lut_per;
  const int L = p->bins, E = L + 1;
  const size_t smem_h = (size_t)(kFusedThreads / 32) * L * sizeof(uint32_t);
  const size_t smem_m = (size_t)((L + 1) & ~1) * 4 + (size_t)L * 8 * 3 + (size_t)E * 8 * 2 + (size_t)E * 8;
  if (!persistent) {
    // compact path: k_hist_part -> k_mid -> k_label_part, PDL-chained
    TSA_CUDA(cudaMemsetAsync(w.counters, 0, sizeof(int32_t) * (2 + 2 * (size_t)p->nz), s));
    a.HC = kCompactHC;
    a.LC = kCompactLC;
    // persistent histogram grid: hist_ctas_per_sm CTAs per SM (measured best: 4,
    // profiles/r1_compact_sweep.log)
    const int hist_per_sm = p->slab_slices > 0 ? p->slab_slices : 4;
    const int hgrid = (int)std::min<int64_t>((int64_t)a.HC * p->nz, (int64_t)hist_per_sm * g_num_sms());
    const int lgrid = (tsa::kSmallLut + 255) / 256;
    a.nlut = lgrid;
    size_t sh = smem_h + 64;
    if (p->slab_slices > 0)  // explicit limit: pad shared memory (keeps ~30 KB for k_mid CTAs)
      sh = std::max(sh, (size_t)(196 * 1024) / (size_t)hist_per_sm);
    const size_t sm = smem_m + 64;
    // the per-slice kernel (its tables need >= kTableThreads threads)
    const int mid_threads = tsa::kMidThreads;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    tsa::k_lut_part<<<lgrid, 256, 0, s>>>(a);
    TSA_TRY(check_cuda("k_lut_part"));
    cfg.gridDim = dim3((unsigned)hgrid);
    cfg.blockDim = dim3(kFusedThreads);
    cfg.dynamicSmemBytes = sh;
    if (p->dtype == TSA_U8) {
      if (sh > 48 * 1024)
        cudaFuncSetAttribute(tsa::k_hist_part<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);
      TSA_CUDA(cudaLaunchKernelEx(&cfg, tsa::k_hist_part<uint8_t>, a));
    } else {
      if (sh > 48 * 1024)
        cudaFuncSetAttribute(tsa::k_hist_part<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);
      TSA_CUDA(cudaLaunchKernelEx(&cfg, tsa::k_hist_part<uint16_t>, a));
    }
    TSA_TRY(check_cuda("k_hist_part"));
    auto mid = p->k == 1 ? (a.mode == tsa::PROD_MAX ? tsa::k_mid<1, tsa::PROD_MAX>
                            : a.mode == tsa::PROD_MIN ? tsa::k_mid<1, tsa::PROD_MIN> : tsa::k_mid<1, tsa::SUM>)
                         : (a.mode == tsa::PROD_MAX ? tsa::k_mid<2, tsa::PROD_MAX>
                            : a.mode == tsa::PROD_MIN ? tsa::k_mid<2, tsa::PROD_MIN> : tsa::k_mid<2, tsa::SUM>);
    if (sm > 48 * 1024) cudaFuncSetAttribute(mid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cfg.gridDim = dim3((unsigned)p->nz);
    cfg.blockDim = dim3((unsigned)mid_threads);
    cfg.dynamicSmemBytes = sm;
    TSA_CUDA(cudaLaunchKernelEx(&cfg, mid, a));
    if (out->labels) {
      cfg.gridDim = dim3((unsigned)a.LC, (unsigned)p->nz);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = 0;
      if (p->dtype == TSA_U8) TSA_CUDA(cudaLaunchKernelEx(&cfg, tsa::k_label_part<uint8_t>, a));
      else TSA_CUDA(cudaLaunchKernelEx(&cfg, tsa::k_label_part<uint16_t>, a));
    }
    return check_cuda("compact path");
  }
  TSA_CUDA(cudaMemsetAsync(w.counters, 0, sizeof(int32_t) * (2 + 2 * (size_t)p->nz), s));
  const size_t smem = std::max(smem_h, smem_m) + 64;
  const int grid = g_num_sms() * 2;
  if (p->dtype == TSA_U8) {
    if (p->k == 1) launch_fused_k<uint8_t, 1>(a, a.mode, smem, grid, s);
    else launch_fused_k<uint8_t, 2>(a, a.mode, smem, grid, s);
  } else {
    if (p->k == 1) launch_fused_k<uint16_t, 1>(a, a.mode, smem, grid, s);
    else launch_fused_k<uint16_t, 2>(a, a.mode, smem, grid, s);
  }
  return check_cuda("k_fused");
}

// k_stream schedule: histogram and label chunks per slice (~256 K voxels
// each; slab_slices overrides), search CTAs per slice, the label lag in
// rounds of the io queue (label_lag overrides) and io CTAs per 4 CTAs.
static void stream_schedule(const tsa_problem *p, int *HC, int *LC, int *SS, int *Dl, int *nio) {
  const int64_t n = p->nx * p->ny;
  const int ch = (int)std::max<int64_t>(1, std::min<int64_t>(64, (n + 262143) / 262144));
  *HC = p->slab_slices > 0 ? p->slab_slices : ch;
  *LC = *HC;
  *SS = 2;
  *Dl = p->label_lag > 0 ? p->label_lag : 32;
  *nio = 2;
}

static tsa_status segment_stream(const tsa_problem *p, const tsa_outputs *out, const SegWs &w,
                                 cudaStream_t s) {
  const int64_t N = p->nx * p->ny, nz = p->nz;
  const int L = p->bins, E = L + 1;
  const bool shannon = p->q == 1.0;
  const int mode = search_mode(p->q, p->objective);
  SearchWs sw;
  Carve c{w.search};
  carve_search(c, sw, nz, N, L, p->k, p->q, p->objective, p->enumeration);
  uint32_t *hist = out->histogram ? out->histogram : w.hist;
  TSA_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * nz * L, s));
  TSA_CUDA(cudaMemsetAsync(w.sctr, 0, sizeof(int32_t) * (3 + tsa::kStCounters * (size_t)nz), s));
  tsa::k_small_luts<<<(tsa::kSmallLut + 255) / 256, 256, 0, s>>>(sw.sp, p->q, shannon);
  TSA_TRY(check_cuda("k_small_luts"));
  const tsa::Luts l = make_luts(p->q, sw.sp);
  tsa::StreamArgs a = {};
  a.vol = reinterpret_cast<const uint8_t *>(p->volume);
  a.n = N;
  a.nz = nz;
  a.L = L;
  a.k = p->k;
  a.hist = hist;
  a.ctr = w.sctr;
  a.status = w.status;
  a.thresholds = out->thresholds;
  a.labels = out->labels;
  a.item_score = w.st_score;
  a.item_key = w.st_key;
  a.NB = stream_tiles(L);
  a.ps = w.ps;
  a.pk = w.pk;
  tsa::ScanArgs &sa = a.scan;
  sa.hist = hist;
  sa.status = w.status;
  sa.nz = nz;
  sa.L = L;
  sa.E = E;
  sa.k = p->k;
  sa.q = p->q;
  sa.shannon = shannon;
  sa.full = 0;
  sa.cC = sw.cC;
  sa.cWhi = sw.cWhi;
  sa.cWlo = sw.cWlo;
  sa.cBin = sw.cBin;
  sa.Asuf = sw.Asuf;
  sa.M = sw.M;
  sa.mmax = nullptr;
  sa.rows = sw.rows;
  sa.RE = k2_row_stride(L);
  sa.luts = l;
  tsa::FinalizeArgs &f = a.fin;
  f.hist = hist;
  f.status_in = w.status;
  f.ps = w.ps;
  f.pk = w.pk;
  f.nparts = 1;
  f.nz = nz;
  f.L = L;
  f.k = p->k;
  f.objective = p->objective;
  f.q = p->q;
  f.thresholds = out->thresholds;
  f.objective_out = out->objective;
  f.status_out = w.status;
  f.status_out2 = out->slice_status;
  stream_schedule(p, &a.HC, &a.LC, &a.SS, &a.Dl, &a.nio);
  a.ltasks = out->labels ? 1 : 0;
  // shared memory: max(H: [L+1] u32 bins + [L] doubles + 1 KB scan scratch,
  //                    L: [L] doubles + [L] ints of the finalize, S: the class-size table)
  const size_t smem_h = 8 * (size_t)((L + 2) / 2 + 1) + 8 * (size_t)L + 1024;
  const size_t smem = std::max({smem_h, (size_t)(L + 1) * 4, (size_t)L * 12, (size_t)tsa::kSN * 16}) + 64;
  auto pick = [&](auto t8) {
    using T = decltype(t8);
    auto f = tsa::k_stream<T, tsa::SUM, 6>;
    if (mode == tsa::PROD_MAX)
      f = l.deg == 5 ? tsa::k_stream<T, tsa::PROD_MAX, 5> : l.deg == 6 ? tsa::k_stream<T, tsa::PROD_MAX, 6>
                                                                     : tsa::k_stream<T, tsa::PROD_MAX, 12>;
    else if (mode == tsa::PROD_MIN)
      f = l.deg == 5 ? tsa::k_stream<T, tsa::PROD_MIN, 5> : l.deg == 6 ? tsa::k_stream<T, tsa::PROD_MIN, 6>
                                                                     : tsa::k_stream<T, tsa::PROD_MIN, 12>;
    return f;
  };
  auto kern = p->dtype == TSA_U8 ? pick(uint8_t{}) : pick(uint16_t{});
  if (smem > 48 * 1024) TSA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  TSA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, tsa::kStThreads, smem));
  const int grid = std::max(1, per_sm) * g_num_sms();
  kern<<<grid, tsa::kStThreads, smem, s>>>(a);
  return check_cuda("k_stream");
}

int32_t tsa_pipeline_kind(const tsa_problem *p) {
  if (tsa_validate(p) != TSA_OK) return 0;
  if (p->pipeline == 3) return stream_eligible(p) ? 3 : -1;
  if (stream_default(p)) return 3;
  if (p->pipeline == 4 || overlap_default(p)) return 4;
  if (p->pipeline < 0 || !fused_eligible(p)) return -1;
  return p->pipeline == 1 ? 1 : 2;
}

size_t tsa_workspace_size(const tsa_problem *p) {
  if (tsa_validate(p) != TSA_OK) return 0;
  return carve_segment(p, nullptr, nullptr);
}

tsa_status tsa_histogram(const tsa_problem *p, uint32_t *hist, int32_t *slice_status, void *stream) {
  TSA_TRY(tsa_validate(p));
  if (!hist || !slice_status) return set_error(TSA_ERR_INVALID_ARG, "hist/slice_status NULL");
  cudaStream_t s = S(stream);
  TSA_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * p->nz * p->bins, s));
  TSA_CUDA(cudaMemsetAsync(slice_status, 0, sizeof(int32_t) * p->nz, s));
  tsa::HistArgs a;
  a.vol = reinterpret_cast<const uint8_t *>(p->volume);
  a.hist = hist;
  a.status = slice_status;
  a.n = p->nx * p->ny;
  a.z0 = 0;
  a.L = p->bins;
  const int threads = 512;
  // privatised copies: one per warp; u16 data with large L packs two 16-bit
  // counters per word (a warp counts < 65536 voxels per launch chunk)
  // (packed 16-bit copies measured 3x slower on 12-bit CT: neighbouring bins
  // share words; kept off -- profiles/r1_c5_histogram.md)
  const bool pack16 = false;
  int reps = pack16 ? std::max(1, std::min(threads / 32, (int)(131072 / (2 * p->bins))))
                    : std::max(1, std::min(threads / 32, (int)(65536 / (4 * p->bins))));
  a.replicas = reps;
  const size_t smem = pack16 ? (size_t)reps * ((p->bins + 1) / 2) * 4 : (size_t)reps * p->bins * 4;
  const int64_t bytes_per_slice = a.n * (p->dtype == TSA_U8 ? 1 : 2);
  // ~64 KB of input per CTA (measured best for 512x512 u8 slices)
  int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(1024, bytes_per_slice / 65536));
  // packed 16-bit counters: a warp must count < 65536 voxels
  if (pack16) chunks = (int)std::max<int64_t>(chunks, (a.n + (threads / 32) * 60000 - 1) / ((threads / 32) * 60000));
  a.chunks = chunks;
  dim3 grid((unsigned)chunks, (unsigned)p->nz);
  if (p->dtype == TSA_U16) {
    // one bin copy + overflow slot; ~128 K voxels (256 KB) per CTA
    a.chunks = (int)std::max<int64_t>(1, std::min<int64_t>(1024, (a.n + 131071) / 131072));
    const size_t sm16 = (size_t)(p->bins + 1) * sizeof(uint32_t);
    tsa::k_hist16<<<dim3((unsigned)a.chunks, (unsigned)p->nz), threads, sm16, s>>>(a);
  } else if (p->dtype == TSA_U8 && p->bins == 256) {
    tsa::k_histogram<uint8_t, false><<<grid, threads, smem, s>>>(a);
  } else if (p->dtype == TSA_U8) {
    tsa::k_histogram<uint8_t, true><<<grid, threads, smem, s>>>(a);
  } else if (pack16) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(tsa::k_histogram_p16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    tsa::k_histogram_p16<<<grid, threads, smem, s>>>(a);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(tsa::k_histogram<uint16_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
    tsa::k_histogram<uint16_t, true><<<grid, threads, smem, s>>>(a);
  }
  return check_cuda("k_histogram");
}

static tsa_status search_impl(const uint32_t *hist, int32_t *slice_status, int64_t nz, int64_t N, int32_t bins,
                              int32_t k, double q, int32_t objective, int32_t enumeration, int32_t units,
                              int32_t unit_begin, int32_t unit_end, double *part_score, uint64_t *part_key,
                              void *workspace, size_t workspace_bytes, void *stream, int k2_ctas_per_sm);

// The k = 2 search (q < 1) skips groups of tuples whose upper bound is below a
// score already reached (exact: k_search.cuh k2_tile PRUNE).  TSA_K2_PRUNE=0
// in the environment runs the plain exhaustive kernel instead (A/B testing).
static bool k2_prune_enabled() {
  const char *e = getenv("TSA_K2_PRUNE");
  return !(e && e[0] == '0');
}
// k_scan_seed (fused) unless TSA_K2_FUSE=0 (k_scan + k_k2_seed; A/B testing)
static bool k2_fuse_enabled() {
  const char *e = getenv("TSA_K2_FUSE");
  return !(e && e[0] == '0');
}

tsa_status tsa_search(const uint32_t *hist, int32_t *slice_status, int64_t nz, int64_t N,
                      int32_t bins, int32_t k, double q, int32_t objective, int32_t enumeration,
                      int32_t units, int32_t unit_begin, int32_t unit_end, double *part_score,
                      uint64_t *part_key, void *workspace, size_t workspace_bytes, void *stream) {
  return search_impl(hist, slice_status, nz, N, bins, k, q, objective, enumeration, units, unit_begin, unit_end,
                     part_score, part_key, workspace, workspace_bytes, stream, 4);
}

static tsa_status search_impl(const uint32_t *hist, int32_t *slice_status, int64_t nz, int64_t N, int32_t bins,
                              int32_t k, double q, int32_t objective, int32_t enumeration, int32_t units,
                              int32_t unit_begin, int32_t unit_end, double *part_score, uint64_t *part_key,
                              void *workspace, size_t workspace_bytes, void *stream, int k2_ctas_per_sm) {
  if (!valid_search_shape(nz, N, bins, k, q, objective, enumeration))
    return set_error(TSA_ERR_INVALID_ARG, "search shape");
  if (!hist || !slice_status || !part_score || !part_key || !workspace)
    return set_error(TSA_ERR_INVALID_ARG, "NULL pointer");
  if (units <= 0) units = tsa_default_units(nz, bins, k, enumeration);
  if (unit_begin < 0 || unit_end > units || unit_begin >= unit_end)
    return set_error(TSA_ERR_INVALID_ARG, "unit range");
  Carve c{reinterpret_cast<char *>(workspace)};
  SearchWs w;
  const size_t need = carve_search(c, w, nz, N, bins, k, q, objective, enumeration);
  if (workspace_bytes < need) return set_error(TSA_ERR_WORKSPACE, "search workspace too small");
  cudaStream_t s = S(stream);
  const bool shannon = q == 1.0;
  const int mode = search_mode(q, objective);
  const tsa::Luts l = make_luts(q, w.sp);
  tsa::k_small_luts<<<(tsa::kSmallLut + 255) / 256, 256, 0, s>>>(w.sp, q, shannon);
  TSA_TRY(check_cuda("k_small_luts"));
  const int E = bins + 1;
  tsa::ScanArgs sa;
  sa.hist = hist;
  sa.status = slice_status;
  sa.nz = nz;
  sa.L = bins;
  sa.E = E;
  sa.k = k;
  sa.q = q;
  sa.shannon = shannon;
  sa.full = enumeration == TSA_ENUM_FULL;
  sa.cC = w.cC;
  sa.cWhi = w.cWhi;
  sa.cWlo = w.cWlo;
  sa.cBin = w.cBin;
  sa.fC = w.fC;
  sa.fWhi = w.fWhi;
  sa.fWlo = w.fWlo;
  sa.fBin = w.fBin;
  sa.Asuf = w.Asuf;
  sa.M = w.M;
  sa.mmax = w.mmax;
  sa.rows = (k == 2 && mode != tsa::SPP) ? w.rows : nullptr;
  sa.RE = k2_row_stride(bins);
  sa.luts = l;
  TSA_CUDA(cudaMemsetAsync(w.counter, 0, 2 * sizeof(int32_t), s));

  // the pruned k = 2 search (q < 1): tables, seed and bound records in one
  // kernel (k_scan_seed); else k_scan (+ k_k2_seed below when unfused)
  // (canonical only: FULL positions include empty bins, where the bound's
  // class-size factor n(a, b0)^-q is undefined for an empty first row)
  const bool k2_prune = k == 2 && mode == tsa::PROD_MAX && enumeration == TSA_ENUM_CANONICAL && k2_prune_enabled();
  const bool fuse_seed = k2_prune && k2_fuse_enabled();
  if (fuse_seed) {
    tsa::SearchArgs ss = {};
    ss.Mz = w.M;
    ss.status = slice_status;
    ss.rows = w.rows;
    ss.RE = k2_row_stride(bins);
    ss.seed = w.seed;
    ss.chk = w.chk;
    ss.nz = nz;
    ss.luts = l;
    const int smem = (int)((size_t)bins * sizeof(double) + 1024 + (size_t)bins * sizeof(uint32_t));
    auto f = l.deg == 5 ? tsa::k_scan_seed<5> : l.deg == 6 ? tsa::k_scan_seed<6> : tsa::k_scan_seed<12>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    f<<<(unsigned)nz, tsa::kTableThreads, (size_t)smem, s>>>(sa, ss, smem);
    TSA_TRY(check_cuda("k_scan_seed"));
  } else {
    switch (mode) {
      case tsa::PROD_MAX: launch_scan<tsa::PROD_MAX>(sa, s); break;
      case tsa::PROD_MIN: launch_scan<tsa::PROD_MIN>(sa, s); break;
      case tsa::SUM: launch_scan<tsa::SUM>(sa, s); break;
      default: launch_scan<tsa::SPP>(sa, s); break;
    }
    TSA_TRY(check_cuda("k_scan"));
  }
  if (enumeration == TSA_ENUM_DP) {
    if (units != 1 || unit_begin != 0 || unit_end != 1)
      return set_error(TSA_ERR_INVALID_ARG, "DP search: one work unit per slice");
    tsa::SearchArgs a = {};
    a.C = w.cC;
    a.Whi = w.cWhi;
    a.Wlo = w.cWlo;
    a.Bin = w.cBin;
    a.Mz = w.M;
    a.status = slice_status;
    a.part_score = part_score;
    a.part_key = part_key;
    a.luts = l;
    a.nz = nz;
    a.E = E;
    a.L = bins;
    // suffix values + the term table (used by slices whose m fits tab_max),
    // within the 227 KB of opt-in shared memory
    const size_t sufb = (size_t)(k + 1) * (bins + 1) * sizeof(double);
    if (sufb > 227 * 1024) return set_error(TSA_ERR_INVALID_ARG, "DP: (k+1)(bins+1) doubles exceed shared memory");
    const size_t tab_max = std::min({tsa::dp_table_bytes(bins), tsa::kDpTableMax, (size_t)227 * 1024 - sufb});
    const size_t smem = sufb + tab_max;
    auto launch_dp = [&](auto kern) -> tsa_status {
      if (smem > 48 * 1024)
        TSA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<(unsigned)nz, 256, smem, s>>>(a, k, tab_max);
      return TSA_OK;
    };
    switch (mode) {
      case tsa::PROD_MAX: TSA_TRY(launch_dp(tsa::k_search_dp<tsa::PROD_MAX>)); break;
      case tsa::PROD_MIN: TSA_TRY(launch_dp(tsa::k_search_dp<tsa::PROD_MIN>)); break;
      default: TSA_TRY(launch_dp(tsa::k_search_dp<tsa::SUM>)); break;
    }
    return check_cuda("k_search_dp");
  }
  const bool full = enumeration == TSA_ENUM_FULL;
  const uint32_t *tC = full ? w.fC : w.cC;
  const double *tWhi = full ? w.fWhi : w.cWhi;
  const double *tWlo = full ? w.fWlo : w.cWlo;
  const int32_t *tBin = full ? w.fBin : w.cBin;
  const bool rt = w.R != nullptr;
  if (rt && !full && mode != tsa::SPP) {
    // canonical k >= 3: tables built per work item by the searching CTA
    // (k_search_tri), shared memory when they fit
    tsa::SearchArgs a = {};
    a.C = w.cC;
    a.Whi = w.cWhi;
    a.Wlo = w.cWlo;
    a.Asuf = w.Asuf;
    a.R = w.R;
    a.PP = w.PP;
    a.AI = w.AI;
    a.counter = w.counter;
    a.Bin = w.cBin;
    a.Mz = w.M;
    a.status = slice_status;
    a.part_score = part_score;
    a.part_key = part_key;
    a.luts = l;
    a.nz = nz;
    a.E = E;
    a.L = bins;
    a.RS = rstride(bins);
    a.units = units;
    a.unit_begin = unit_begin;
    a.nunits = unit_end - unit_begin;
    // CTAs sharing a slice: with the exact bounds most items are dropped
    // cheaply, so fewer table copies win (profiles/r2zq: c3 ss 1/2/4 = 283/288/309
    // us, c4 ss 2/4/8 = 221/232/251 us)
    a.ss = k == 3 ? 1 : 2;
    if (const char *e = getenv("TSA_TRI_SS")) a.ss = std::max(1, std::min(kTriSS, atoi(e)));  // A/B
    a.TS = tsa::tri_slice_stride(bins);
    a.ccur = w.ccur;
    a.item_score = w.item_score;
    a.item_key = w.item_key;
    TSA_CUDA(cudaMemsetAsync(w.ccur, 0, sizeof(int32_t) * nz, s));
    const int64_t items = nz * (int64_t)a.ss;
    const size_t smem = tsa::kTriSmemBytes;
    auto kern = k == 3 ? (mode == tsa::PROD_MAX ? tsa::k_search_tri<3, tsa::PROD_MAX>
                          : mode == tsa::PROD_MIN ? tsa::k_search_tri<3, tsa::PROD_MIN> : tsa::k_search_tri<3, tsa::SUM>)
                       : (mode == tsa::PROD_MAX ? tsa::k_search_tri<4, tsa::PROD_MAX>
                          : mode == tsa::PROD_MIN ? tsa::k_search_tri<4, tsa::PROD_MIN> : tsa::k_search_tri<4, tsa::SUM>);
    TSA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    auto tab = k == 3 ? (mode == tsa::PROD_MAX ? tsa::k_tri_tables<3, tsa::PROD_MAX>
                         : mode == tsa::PROD_MIN ? tsa::k_tri_tables<3, tsa::PROD_MIN> : tsa::k_tri_tables<3, tsa::SUM>)
                      : (mode == tsa::PROD_MAX ? tsa::k_tri_tables<4, tsa::PROD_MAX>
                         : mode == tsa::PROD_MIN ? tsa::k_tri_tables<4, tsa::PROD_MIN> : tsa::k_tri_tables<4, tsa::SUM>);
    tab<<<(unsigned)nz, 256, 0, s>>>(a);  // per-slice tables and seed, once
    // (building them in 104 KB of shared memory with a CTA-wide seed measured
    // slower: 96 vs 46 us on c3)
    TSA_TRY(check_cuda("k_tri_tables"));
    const unsigned grid = (unsigned)std::min<int64_t>(items, 2 * g_num_sms());
    // TSA_TRI_STAGE=0 (A/B): no shared-memory copy of the slice's tables, the
    // search reads them through L1/L2 (with the exact bounds most of them are
    // never read)
    const char *st_env = getenv("TSA_TRI_STAGE");
    const bool stage = !(st_env && st_env[0] == '0');
    kern<<<grid, 256, stage ? smem : 0, s>>>(a, stage ? (int)(smem / sizeof(double)) : 0);
    TSA_TRY(check_cuda("k_search_tri"));
    tsa::k_fold_slots<<<(unsigned)((nz + 7) / 8), 256, 0, s>>>(w.item_score, w.item_key, a.ss, nz, a.nunits,
                                                              part_score, part_key);
    return check_cuda("k_fold_slots");
  }
  if (rt) {
    switch (mode) {
      case tsa::PROD_MAX: launch_rtable<tsa::PROD_MAX>(w, tC, tWhi, tWlo, slice_status, nz, E, bins, l, s); break;
      case tsa::PROD_MIN: launch_rtable<tsa::PROD_MIN>(w, tC, tWhi, tWlo, slice_status, nz, E, bins, l, s); break;
      default: launch_rtable<tsa::SUM>(w, tC, tWhi, tWlo, slice_status, nz, E, bins, l, s); break;
    }
    TSA_TRY(check_cuda("k_rtable"));
  }
  tsa::SearchArgs a;
  a.C = tC;
  a.Whi = tWhi;
  a.Wlo = tWlo;
  a.Asuf = w.Asuf;
  a.R = w.R;
  a.PP = w.PP;
  a.AI = w.AI;
  a.counter = w.counter;
  a.Bin = tBin;
  a.Mz = w.M;
  a.status = slice_status;
  a.part_score = part_score;
  a.part_key = part_key;
  a.luts = l;
  a.nz = nz;
  a.E = E;
  a.L = bins;
  a.RS = rstride(bins);
  a.units = units;
  a.unit_begin = unit_begin;
  a.nunits = unit_end - unit_begin;
  a.mmax = w.mmax;
  a.item_score = w.item_score;
  a.item_key = w.item_key;
  a.rows = w.rows;
  a.RE = k2_row_stride(bins);
  a.seed = w.seed;
  a.chk = w.chk;
  if (k == 2 && mode != tsa::SPP) {
    // warp-per-a-block search from a global item queue, then the per-unit fold
    const int grid = k2_ctas_per_sm * g_num_sms();
    auto kern = tsa::k_search_k2<tsa::SUM, 6>;
    if (k2_prune) {
      // seed scores (unless k_scan_seed made them), then the bounded search
      // (bit-identical result, k_search.cuh k2_tile PRUNE)
      if (!fuse_seed) {
        auto sk = l.deg == 5 ? tsa::k_k2_seed<tsa::PROD_MAX, 5> : l.deg == 6 ? tsa::k_k2_seed<tsa::PROD_MAX, 6>
                                                                            : tsa::k_k2_seed<tsa::PROD_MAX, 12>;
        sk<<<(unsigned)nz, 256, 0, s>>>(a);
        TSA_TRY(check_cuda("k_k2_seed"));
      }
      kern = l.deg == 5   ? tsa::k_search_k2<tsa::PROD_MAX, 5, true>
             : l.deg == 6 ? tsa::k_search_k2<tsa::PROD_MAX, 6, true>
                          : tsa::k_search_k2<tsa::PROD_MAX, 12, true>;
    } else if (mode == tsa::PROD_MAX)
      kern = l.deg == 5 ? tsa::k_search_k2<tsa::PROD_MAX, 5> : l.deg == 6 ? tsa::k_search_k2<tsa::PROD_MAX, 6>
                                                                          : tsa::k_search_k2<tsa::PROD_MAX, 12>;
    else if (mode == tsa::PROD_MIN)
      kern = l.deg == 5 ? tsa::k_search_k2<tsa::PROD_MIN, 5> : l.deg == 6 ? tsa::k_search_k2<tsa::PROD_MIN, 6>
                                                                          : tsa::k_search_k2<tsa::PROD_MIN, 12>;
    kern<<<grid, 256, 0, s>>>(a);  // (slice-per-CTA with the rows in shared memory measured slower: 664 vs 575 us)
    TSA_TRY(check_cuda("k_search_k2"));
    const int64_t nt = nz * (int64_t)a.nunits;
    tsa::k_merge_items<<<(unsigned)((nt + 7) / 8), 256, 0, s>>>(w.item_score, w.item_key, w.M, slice_status, w.mmax,
                                                                  nz, units, unit_begin, a.nunits, part_score,
                                                                  part_key);
    return check_cuda("k_merge_items");
  }
  dim3 grid((unsigned)(unit_end - unit_begin), (unsigned)nz);
  switch (mode) {
    case tsa::PROD_MAX: launch_search_mode<tsa::PROD_MAX>(k, a, grid, s, rt); break;
    case tsa::PROD_MIN: launch_search_mode<tsa::PROD_MIN>(k, a, grid, s, rt); break;
    case tsa::SUM: launch_search_mode<tsa::SUM>(k, a, grid, s, rt); break;
    default: launch_search_mode<tsa::SPP>(k, a, grid, s, false); break;
  }
  return check_cuda("k_search");
}

size_t tsa_class_consts_workspace_size(void) { return (size_t)tsa::kSmallLut * sizeof(double); }

tsa_status tsa_class_consts(const uint32_t *n, int64_t count, double q, double *a, double *b,
                            void *workspace, size_t workspace_bytes, void *stream) {
  if (!n || !a || count < 0 || !(q > 0.0) || !std::isfinite(q) || !workspace)
    return set_error(TSA_ERR_INVALID_ARG, "class_consts args");
  if (workspace_bytes < tsa_class_consts_workspace_size())
    return set_error(TSA_ERR_WORKSPACE, "class_consts workspace too small");
  cudaStream_t s = S(stream);
  double *sp = reinterpret_cast<double *>(workspace);
  tsa::k_small_luts<<<(tsa::kSmallLut + 255) / 256, 256, 0, s>>>(sp, q, q == 1.0);
  if (count > 0) {
    const int64_t blocks = std::min<int64_t>((count + 255) / 256, 8 * g_num_sms());
    tsa::k_class_consts<<<(unsigned)blocks, 256, 0, s>>>(n, count, make_luts(q, sp), a, b);
  }
  return check_cuda("k_class_consts");
}

tsa_status tsa_merge(const double *part_score, const uint64_t *part_key, int32_t nparts,
                     int64_t nz, double *score, uint64_t *key, void *stream) {
  if (!part_score || !part_key || !score || !key || nparts <= 0 || nz <= 0)
    return set_error(TSA_ERR_INVALID_ARG, "merge args");
  const int warps = 4;
  tsa::k_merge<<<(unsigned)((nz + warps - 1) / warps), 32 * warps, 0, S(stream)>>>(
      part_score, part_key, nparts, nz, score, key);
  return check_cuda("k_merge");
}

// The staged step's split finalize (k_decide + labels + k_finalize_phi as the
// labels' PDL dependent) unless TSA_SPLIT_FINALIZE=0 (A/B testing); the label
// kernel uses TSA_LABEL_CTAS (default 8) CTAs per SM (c5 A/B, profiles/r2zi:
// 8 -> 1.197 ms, 7 -> 1.205, 6 -> 1.221, unsplit 1.207).
static bool split_finalize_enabled() {
  const char *e = getenv("TSA_SPLIT_FINALIZE");
  return !(e && e[0] == '0');
}
static int label_ctas_split() {
  const char *e = getenv("TSA_LABEL_CTAS");
  const int v = e ? atoi(e) : 8;
  return v >= 1 && v <= 8 ? v : 8;
}

static tsa::FinalizeArgs finalize_args(const uint32_t *hist, const int32_t *status_in, int64_t nz, int32_t bins,
                                       int32_t k, double q, int32_t objective, const double *ps,
                                       const uint64_t *pk, int32_t nparts, int32_t *thresholds,
                                       double *objective_out, int32_t *status_out, int32_t *status_out2) {
  tsa::FinalizeArgs f;
  f.hist = hist;
  f.status_in = status_in;
  f.ps = ps;
  f.pk = pk;
  f.nparts = nparts;
  f.nz = nz;
  f.L = bins;
  f.k = k;
  f.objective = objective;
  f.q = q;
  f.thresholds = thresholds;
  f.objective_out = objective_out;
  f.status_out = status_out;
  f.status_out2 = status_out2;
  return f;
}

static tsa_status decide_impl(const uint32_t *hist, const int32_t *status_in, int64_t nz, int32_t bins,
                              int32_t k, double q, int32_t objective, const double *ps, const uint64_t *pk,
                              int32_t nparts, int32_t *thresholds, int32_t *status_out, int32_t *status_out2,
                              cudaStream_t s) {
  const tsa::FinalizeArgs f = finalize_args(hist, status_in, nz, bins, k, q, objective, ps, pk, nparts,
                                            thresholds, nullptr, status_out, status_out2);
  tsa::k_decide<<<(unsigned)((nz + 7) / 8), 256, 0, s>>>(f);
  return check_cuda("k_decide");
}

static tsa_status finalize_impl(const uint32_t *hist, const int32_t *status_in, int64_t nz,
                                int32_t bins, int32_t k, double q, int32_t objective,
                                const double *ps, const uint64_t *pk, int32_t nparts,
                                int32_t *thresholds, double *objective_out, int32_t *status_out,
                                int32_t *status_out2, cudaStream_t s, bool phi_pdl = false) {
  if (phi_pdl) {  // k_finalize_phi as the PDL dependent of the label kernel just launched
    const tsa::FinalizeArgs f = finalize_args(hist, status_in, nz, bins, k, q, objective, ps, pk, nparts,
                                              thresholds, objective_out, nullptr, nullptr);
    const size_t smem = (size_t)bins * (sizeof(double) + sizeof(int));
    if (smem > 32 * 1024)
      cudaFuncSetAttribute(tsa::k_finalize_phi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3((unsigned)nz);
    cfg.blockDim = dim3(tsa::kFinThreads);
    cfg.dynamicSmemBytes = smem;
    TSA_CUDA(cudaLaunchKernelEx(&cfg, tsa::k_finalize_phi, f));
    return check_cuda("k_finalize_phi");
  }
  tsa::FinalizeArgs f;
  f.hist = hist;
  f.status_in = status_in;
  f.ps = ps;
  f.pk = pk;
  f.nparts = nparts;
  f.nz = nz;
  f.L = bins;
  f.k = k;
  f.objective = objective;
  f.q = q;
  f.thresholds = thresholds;
  f.objective_out = objective_out;
  f.status_out = status_out;
  f.status_out2 = status_out2;
  const size_t smem = (size_t)bins * (sizeof(double) + sizeof(int));
  if (smem > 32 * 1024)
    cudaFuncSetAttribute(tsa::k_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tsa::k_finalize<<<(unsigned)nz, tsa::kFinThreads, smem, s>>>(f);
  return check_cuda("k_finalize");
}

tsa_status tsa_finalize(const uint32_t *hist, const int32_t *slice_status, int64_t nz,
                        int32_t bins, int32_t k, double q, int32_t objective,
                        const double *part_score, const uint64_t *part_key, int32_t nparts,
                        const tsa_outputs *out, void *stream) {
  if (!valid_search_shape(nz, 1, bins, k, q, objective, TSA_ENUM_CANONICAL))
    return set_error(TSA_ERR_INVALID_ARG, "finalize shape");
  if (!hist || !slice_status || !part_score || !part_key || nparts <= 0 || !out ||
      !out->thresholds)
    return set_error(TSA_ERR_INVALID_ARG, "finalize pointers");
  return finalize_impl(hist, slice_status, nz, bins, k, q, objective, part_score, part_key,
                       nparts, out->thresholds, out->objective, out->slice_status, nullptr, S(stream));
}

static tsa_status label_impl(const tsa_problem *p, const int32_t *thresholds, const int32_t *slice_status,
                             uint8_t *labels, void *stream, int ctas_per_sm);

tsa_status tsa_label(const tsa_problem *p, const int32_t *thresholds, const int32_t *slice_status,
                     uint8_t *labels, void *stream) {
  return label_impl(p, thresholds, slice_status, labels, stream, 8);
}

// ctas_per_sm: the grid-stride label kernel's CTAs per SM (8 = every warp
// slot; the overlap pipeline leaves room for the concurrent search)
static tsa_status label_impl(const tsa_problem *p, const int32_t *thresholds, const int32_t *slice_status,
                             uint8_t *labels, void *stream, int ctas_per_sm) {
  TSA_TRY(tsa_validate(p));
  if (!thresholds || !labels) return set_error(TSA_ERR_INVALID_ARG, "label pointers");
  tsa::LabelArgs a;
  a.vol = reinterpret_cast<const uint8_t *>(p->volume);
  a.labels = labels;
  a.thr = thresholds;
  a.status = slice_status;
  a.n = p->nx * p->ny;
  a.z0 = 0;
  a.z1 = p->nz;
  a.k = p->k;
  const bool aligned = a.n % 16 == 0 && (reinterpret_cast<uintptr_t>(p->volume) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(labels) & 15) == 0;
  if (aligned) {
    const int64_t groups = a.n / 16 * p->nz;
    const int64_t blocks = std::min<int64_t>((groups + 255) / 256, (int64_t)g_num_sms() * ctas_per_sm);
    cudaStream_t s = S(stream);
    if (p->dtype == TSA_U8) {
      switch (p->k) {
        case 1: tsa::k_label_flat<uint8_t, 1><<<(unsigned)blocks, 256, 0, s>>>(a); break;
        case 2: tsa::k_label_flat<uint8_t, 2><<<(unsigned)blocks, 256, 0, s>>>(a); break;
        case 3: tsa::k_label_flat<uint8_t, 3><<<(unsigned)blocks, 256, 0, s>>>(a); break;
        default: tsa::k_label_flat<uint8_t, 4><<<(unsigned)blocks, 256, 0, s>>>(a); break;
      }
    } else {
      switch (p->k) {
        case 1: tsa::k_label_flat<uint16_t, 1><<<(unsigned)blocks, 256, 0, s>>>(a); break;
        case 2: tsa::k_label_flat<uint16_t, 2><<<(unsigned)blocks, 256, 0, s>>>(a); break;
        case 3: tsa::k_label_flat<uint16_t, 3><<<(unsigned)blocks, 256, 0, s>>>(a); break;
        default: tsa::k_label_flat<uint16_t, 4><<<(unsigned)blocks, 256, 0, s>>>(a); break;
      }
    }
  } else {
    const int64_t cx = std::max<int64_t>(1, std::min<int64_t>(64, a.n / 4096));
    dim3 grid((unsigned)cx, (unsigned)p->nz);
    if (p->dtype == TSA_U8)
      tsa::k_label_generic<uint8_t><<<grid, 256, 0, S(stream)>>>(a);
    else
      tsa::k_label_generic<uint16_t><<<grid, 256, 0, S(stream)>>>(a);
  }
  return check_cuda("k_label");
}

// Overlap pipeline (pipeline = 4): the staged kernels on slabs of slices over
// two streams -- the caller's stream runs the HBM-bound histogram of slab c+1
// and the labels of slab c-1 while a second stream (created by this call and
// released at its end) runs the FP64-bound tables / search / finalize of slab
// c on half of each SM (two search CTAs per SM), so the two kinds of work
// overlap.  Same kernels, same partition of the tuple space: bit-identical
// to the staged pipeline.  Not used while `stream` is being captured (the
// extra stream would outlive the capture): staged instead.
// label CTAs per SM inside the overlap pipeline (TSA_OVL_LABEL_CTAS, A/B)
static int ovl_label_ctas() {
  const char *e = getenv("TSA_OVL_LABEL_CTAS");
  const int v = e ? atoi(e) : 4;
  return v >= 1 && v <= 8 ? v : 4;
}
// k = 2 search CTAs per SM inside the overlap pipeline (TSA_OVL_SEARCH_CTAS, A/B)
static int ovl_search_ctas() {
  const char *e = getenv("TSA_OVL_SEARCH_CTAS");
  const int v = e ? atoi(e) : 2;
  return v >= 1 && v <= 4 ? v : 2;
}
static tsa_status label_impl(const tsa_problem *p, const int32_t *thresholds, const int32_t *slice_status,
                             uint8_t *labels, void *stream, int ctas_per_sm);

static tsa_status segment_overlap(const tsa_problem *p, const tsa_outputs *out, const SegWs &w, cudaStream_t s) {
  const int64_t nz = p->nz, n = p->nx * p->ny;
  const size_t esz = p->dtype == TSA_U8 ? 1 : 2;
  const int G0 = (int)std::min<int64_t>({nz, (int64_t)64, p->slab_slices > 0 ? (int64_t)p->slab_slices : 8});
  const int64_t cz = (nz + G0 - 1) / G0;  // slices per slab
  const int G = (int)((nz + cz - 1) / cz);  // slabs (no empty one)
  uint32_t *hist = out->histogram ? out->histogram : w.hist;
  cudaStream_t a = nullptr;
  TSA_CUDA(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
  cudaEvent_t ev[2 * 64 + 1];
  const int nev = 2 * G + 1;
  for (int i = 0; i < nev; i++) TSA_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  cudaEvent_t e_start = ev[0], *e_h = ev + 1, *e_s = ev + 1 + G;
  tsa_status rc = TSA_OK;
  auto sub = [&](int c, tsa_problem *q, int64_t *z0) {
    *q = *p;
    *z0 = (int64_t)c * cz;
    q->nz = std::min(cz, nz - *z0);
    q->volume = reinterpret_cast<const char *>(p->volume) + (size_t)(*z0) * n * esz;
  };
  auto label = [&](int c) -> tsa_status {
    tsa_problem q;
    int64_t z0;
    sub(c, &q, &z0);
    if (cudaStreamWaitEvent(s, e_s[c], 0) != cudaSuccess) return set_error(TSA_ERR_CUDA, "overlap: wait search");
    if (!out->labels) return TSA_OK;
    return label_impl(&q, out->thresholds + z0 * p->k, w.status + z0, out->labels + (size_t)z0 * n, s,
                      ovl_label_ctas());
  };
  if (cudaEventRecord(e_start, s) != cudaSuccess || cudaStreamWaitEvent(a, e_start, 0) != cudaSuccess)
    rc = set_error(TSA_ERR_CUDA, "overlap: fork");
  for (int c = 0; c < G && rc == TSA_OK; c++) {
    tsa_problem q;
    int64_t z0;
    sub(c, &q, &z0);
    rc = tsa_histogram(&q, hist + z0 * p->bins, w.status + z0, s);
    if (rc == TSA_OK && (cudaEventRecord(e_h[c], s) != cudaSuccess || cudaStreamWaitEvent(a, e_h[c], 0) != cudaSuccess))
      rc = set_error(TSA_ERR_CUDA, "overlap: histogram event");
    const int32_t U = units_of(&q);
    if (rc == TSA_OK)
      rc = search_impl(hist + z0 * p->bins, w.status + z0, q.nz, n, p->bins, p->k, p->q, p->objective,
                       p->enumeration, U, 0, U, w.ps, w.pk, w.search, w.search_bytes, a, ovl_search_ctas());
    if (rc == TSA_OK)
      rc = finalize_impl(hist + z0 * p->bins, w.status + z0, q.nz, p->bins, p->k, p->q, p->objective, w.ps, w.pk,
                         U, out->thresholds + z0 * p->k, out->objective ? out->objective + z0 : nullptr,
                         w.status + z0, out->slice_status ? out->slice_status + z0 : nullptr, a);
    if (rc == TSA_OK && cudaEventRecord(e_s[c], a) != cudaSuccess) rc = set_error(TSA_ERR_CUDA, "overlap: search event");
    if (rc == TSA_OK && c > 0) rc = label(c - 1);
  }
  if (rc == TSA_OK) rc = label(G - 1);  // also joins the second stream into `s`
  for (int i = 0; i < nev; i++) cudaEventDestroy(ev[i]);
  cudaStreamDestroy(a);  // released once its queued work is done
  return rc;
}

tsa_status tsa_segment(const tsa_problem *p, const tsa_outputs *out, void *workspace,
                       size_t workspace_bytes, void *stream) {
  TSA_TRY(tsa_validate(p));
  if (!out || !out->thresholds) return set_error(TSA_ERR_INVALID_ARG, "outputs->thresholds NULL");
  if (!workspace) return set_error(TSA_ERR_INVALID_ARG, "workspace NULL");
  SegWs w;
  const size_t need = carve_segment(p, reinterpret_cast<char *>(workspace), &w);
  if (workspace_bytes < need) return set_error(TSA_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = S(stream);
  const bool labels_aligned = !out->labels || (reinterpret_cast<uintptr_t>(out->labels) & 15) == 0;
  if ((p->pipeline == 3 || stream_default(p)) && stream_eligible(p) && labels_aligned)
    return segment_stream(p, out, w, s);
  if (p->pipeline == 3) return set_error(TSA_ERR_INVALID_ARG, "stream pipeline requested but the problem is not eligible");
  if (p->pipeline >= 0 && p->pipeline <= 2 && fused_eligible(p) && labels_aligned)
    return segment_fused(p, out, w, s, p->pipeline == 1);
  if (p->pipeline == 4 || overlap_default(p)) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    TSA_CUDA(cudaStreamIsCapturing(s, &cs));
    if (cs == cudaStreamCaptureStatusNone) return segment_overlap(p, out, w, s);
  }
  if (p->pipeline > 0 && p->pipeline != 4)
    return set_error(TSA_ERR_INVALID_ARG, "fused/compact pipeline requested but the problem is not eligible");
  uint32_t *hist = out->histogram ? out->histogram : w.hist;
  const int32_t U = units_of(p);
  TSA_TRY(tsa_histogram(p, hist, w.status, stream));
  TSA_TRY(tsa_search(hist, w.status, p->nz, p->nx * p->ny, p->bins, p->k, p->q, p->objective,
                     p->enumeration, U, 0, U, w.ps, w.pk, w.search, w.search_bytes, stream));
  if (out->labels && out->objective && split_finalize_enabled()) {
    // k_decide -> labels -> k_finalize_phi (PDL dependent of the labels, next
    // to them on the SMs; k_finalize.cuh)
    TSA_TRY(decide_impl(hist, w.status, p->nz, p->bins, p->k, p->q, p->objective, w.ps, w.pk, U,
                        out->thresholds, w.status, out->slice_status, s));
    TSA_TRY(label_impl(p, out->thresholds, w.status, out->labels, stream, label_ctas_split()));
    return finalize_impl(hist, w.status, p->nz, p->bins, p->k, p->q, p->objective, w.ps, w.pk, U,
                         out->thresholds, out->objective, nullptr, nullptr, s, true);
  }
  TSA_TRY(finalize_impl(hist, w.status, p->nz, p->bins, p->k, p->q, p->objective, w.ps, w.pk, U,
                        out->thresholds, out->objective, w.status, out->slice_status, s));
  if (out->labels) TSA_TRY(tsa_label(p, out->thresholds, w.status, out->labels, stream));
  return TSA_OK;
}

// ------------------------------------------------------------ q sweep
// Staged path per q (the same kernels as tsa_segment's staged pipeline), the
// histogram once.  Layout: [status of the histogram pass][staged workspace for
// the largest per-q size].
static bool sweep_args_ok(const tsa_problem *p, const double *qs, int32_t nq) {
  if (!p || !qs || nq < 1 || nq > 64) return false;
  for (int i = 0; i < nq; i++) {
    tsa_problem pq = *p;
    pq.q = qs[i];
    pq.pipeline = -1;
    if (tsa_validate(&pq) != TSA_OK) return false;
  }
  return true;
}

// q values in flight at once (kSweepLanes streams, a staged workspace slot
// each): the per-q chains are latency-bound kernels of ~one wave each, so
// running several side by side fills the GPU (round 2).
constexpr int kSweepLanes = 4;
static size_t sweep_slot_bytes(const tsa_problem *p, const double *qs, int32_t nq) {
  size_t mx = 0;
  for (int i = 0; i < nq; i++) {
    tsa_problem pq = *p;
    pq.q = qs[i];
    pq.pipeline = -1;
    mx = std::max(mx, carve_segment(&pq, nullptr, nullptr));
  }
  return align_up(mx);
}

size_t tsa_sweep_workspace_size(const tsa_problem *p, const double *qs, int32_t nq) {
  if (!sweep_args_ok(p, qs, nq)) return 0;
  return align_up((size_t)p->nz * sizeof(int32_t)) +
         (size_t)std::min<int32_t>(nq, kSweepLanes) * sweep_slot_bytes(p, qs, nq);
}

tsa_status tsa_segment_sweep(const tsa_problem *p, const double *qs, int32_t nq,
                             const tsa_outputs *outs, void *workspace, size_t workspace_bytes,
                             void *stream) {
  if (!sweep_args_ok(p, qs, nq)) return set_error(TSA_ERR_INVALID_ARG, "sweep: problem or q values");
  if (!outs || !workspace) return set_error(TSA_ERR_INVALID_ARG, "sweep: outputs / workspace NULL");
  for (int i = 0; i < nq; i++)
    if (!outs[i].thresholds) return set_error(TSA_ERR_INVALID_ARG, "sweep: outputs[i].thresholds NULL");
  const size_t need = tsa_sweep_workspace_size(p, qs, nq);
  if (workspace_bytes < need) return set_error(TSA_ERR_WORKSPACE, "sweep workspace too small");
  cudaStream_t s = S(stream);
  Carve c{reinterpret_cast<char *>(workspace)};
  int32_t *hstatus = c.take<int32_t>((size_t)p->nz);
  char *rest = c.take<char>(0);
  SegWs w;
  carve_segment(p, rest, &w);
  uint32_t *hist = w.hist;
  for (int i = 0; i < nq; i++)
    if (outs[i].histogram) {
      hist = outs[i].histogram;
      break;
    }
  TSA_TRY(tsa_histogram(p, hist, hstatus, stream));
  // one label pass for all q (k_label_sweep) when the buffers allow vector I/O
  bool sweep_labels = (p->nx * p->ny) % 16 == 0 && (reinterpret_cast<uintptr_t>(p->volume) & 15) == 0;
  for (int i = 0; i < nq; i++)
    if (outs[i].labels && (reinterpret_cast<uintptr_t>(outs[i].labels) & 15) != 0) sweep_labels = false;
  for (int i = 0; i < nq; i++)
    if (outs[i].histogram && outs[i].histogram != hist)
      TSA_CUDA(cudaMemcpyAsync(outs[i].histogram, hist, sizeof(uint32_t) * p->nz * p->bins,
                               cudaMemcpyDeviceToDevice, s));
  // q chains on up to kSweepLanes streams (q i on lane i % lanes, slot i % lanes
  // of the workspace; the caller's stream is lane 0); one lane while `stream`
  // is being captured (the extra streams would outlive the capture)
  const size_t slot = sweep_slot_bytes(p, qs, nq);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  TSA_CUDA(cudaStreamIsCapturing(s, &cs));
  int lanes = cs == cudaStreamCaptureStatusNone ? std::min<int32_t>(nq, kSweepLanes) : 1;
  if (const char *e = getenv("TSA_SWEEP_LANES")) lanes = std::max(1, std::min(lanes, atoi(e)));  // A/B
  cudaStream_t ls[kSweepLanes] = {s};
  cudaEvent_t ev[kSweepLanes] = {};
  tsa_status rc = TSA_OK;
  for (int j = 0; j < lanes && rc == TSA_OK; j++) {
    if (cudaEventCreateWithFlags(&ev[j], cudaEventDisableTiming) != cudaSuccess) rc = set_error(TSA_ERR_CUDA, "sweep: event");
    if (j > 0 && rc == TSA_OK && cudaStreamCreateWithFlags(&ls[j], cudaStreamNonBlocking) != cudaSuccess)
      rc = set_error(TSA_ERR_CUDA, "sweep: stream");
  }
  if (rc == TSA_OK && lanes > 1) {  // fork after the histogram
    if (cudaEventRecord(ev[0], s) != cudaSuccess) rc = set_error(TSA_ERR_CUDA, "sweep: fork");
    for (int j = 1; j < lanes && rc == TSA_OK; j++)
      if (cudaStreamWaitEvent(ls[j], ev[0], 0) != cudaSuccess) rc = set_error(TSA_ERR_CUDA, "sweep: fork");
  }
  for (int i = 0; i < nq && rc == TSA_OK; i++) {
    const int j = i % lanes;
    cudaStream_t sj = ls[j];
    tsa_problem pq = *p;
    pq.q = qs[i];
    SegWs wq;
    carve_segment(&pq, rest + (size_t)j * slot, &wq);
    const int32_t U = units_of(&pq);
    if (cudaMemcpyAsync(wq.status, hstatus, sizeof(int32_t) * p->nz, cudaMemcpyDeviceToDevice, sj) != cudaSuccess) {
      rc = set_error(TSA_ERR_CUDA, "sweep: status copy");
      break;
    }
    rc = tsa_search(hist, wq.status, pq.nz, pq.nx * pq.ny, pq.bins, pq.k, pq.q, pq.objective, pq.enumeration, U, 0,
                    U, wq.ps, wq.pk, wq.search, wq.search_bytes, sj);
    if (rc == TSA_OK)
      rc = finalize_impl(hist, wq.status, pq.nz, pq.bins, pq.k, pq.q, pq.objective, wq.ps, wq.pk, U,
                         outs[i].thresholds, outs[i].objective, wq.status, outs[i].slice_status, sj);
    if (rc == TSA_OK && outs[i].labels && !sweep_labels)
      rc = tsa_label(&pq, outs[i].thresholds, wq.status, outs[i].labels, sj);
  }
  for (int j = 1; j < lanes; j++) {  // join (also on errors: leave no lane behind)
    if (ls[j] && ev[j] && cudaEventRecord(ev[j], ls[j]) == cudaSuccess) cudaStreamWaitEvent(s, ev[j], 0);
  }
  for (int j = 0; j < lanes; j++) {
    if (ev[j]) cudaEventDestroy(ev[j]);
    if (j > 0 && ls[j]) cudaStreamDestroy(ls[j]);  // released once its queued work is done
  }
  TSA_TRY(rc);
  if (sweep_labels) {  // every q's labels from one read of the volume
    for (int q0 = 0; q0 < nq; q0 += tsa::kSweepMaxQ) {
      tsa::LabelSweepArgs la = {};
      la.vol = reinterpret_cast<const uint8_t *>(p->volume);
      la.n = p->nx * p->ny;
      la.k = p->k;
      for (int i = q0; i < std::min(nq, q0 + tsa::kSweepMaxQ); i++) {
        if (!outs[i].labels) continue;
        la.thr[la.nq] = outs[i].thresholds;
        la.lab[la.nq] = outs[i].labels;
        la.nq++;
      }
      if (la.nq == 0) continue;
      const int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(64, la.n / 16 / 2048));
      const dim3 grid((unsigned)chunks, (unsigned)p->nz);
      auto kern = p->dtype == TSA_U8
                      ? (p->k == 1 ? tsa::k_label_sweep<uint8_t, 1> : p->k == 2 ? tsa::k_label_sweep<uint8_t, 2>
                         : p->k == 3 ? tsa::k_label_sweep<uint8_t, 3> : tsa::k_label_sweep<uint8_t, 4>)
                      : (p->k == 1 ? tsa::k_label_sweep<uint16_t, 1> : p->k == 2 ? tsa::k_label_sweep<uint16_t, 2>
                         : p->k == 3 ? tsa::k_label_sweep<uint16_t, 3> : tsa::k_label_sweep<uint16_t, 4>);
      kern<<<grid, 256, 0, s>>>(la);
      TSA_TRY(check_cuda("k_label_sweep"));
    }
  }
  return TSA_OK;
}

// ------------------------------------------------------------------- 2-D
}  // extern "C"

static bool valid2d(const tsa2d_problem *p) {
  return p && p->volume && p->nx > 0 && p->ny > 0 && p->nz > 0 && p->nz <= 65535 && p->nx <= 65535 &&
         p->nx * p->ny < (int64_t(1) << 31) && p->bins >= 2 && p->bins <= 256 && p->q > 0.0 &&
         std::isfinite(p->q) && (p->cluster == 0 || (p->cluster >= 4 && p->cluster <= 8));
}

constexpr size_t kSmem2dMax = 227 * 1024;  // opt-in shared memory per CTA (sm_100a)

struct Plan2d {
  int CL, R, LP, rr, rounds;
  size_t smem;
};

static Plan2d plan2d(const tsa2d_problem *p) {
  Plan2d pl;
  pl.LP = (p->bins + 1) & ~1;
  // smallest cluster whose CTAs each count <= 65536 pixels in one round (a
  // single round of exactly 65536 handles the one counter that can wrap)
  int CL = p->cluster;
  if (CL == 0) {
    CL = 8;
    for (int c = 4; c <= 8; c++)
      if (((p->ny + c - 1) / c) * p->nx <= 65536) {
        CL = c;
        break;
      }
  }
  // shared-memory fit (the L x L private histogram plus the band tables)
  while (p->cluster == 0 && CL < 8 &&
         tsa::smem2d_layout(p->bins, pl.LP, (p->bins + CL - 1) / CL).total > kSmem2dMax)
    CL++;
  pl.CL = CL;
  pl.R = (p->bins + CL - 1) / CL;
  const int64_t rows_max = (p->ny + CL - 1) / CL;
  pl.rr = rows_max * p->nx <= 65536 ? (int)rows_max : (int)std::max<int64_t>(1, 65535 / p->nx);
  pl.rounds = (int)((rows_max + pl.rr - 1) / pl.rr);
  pl.smem = tsa::smem2d_layout(p->bins, pl.LP, pl.R).total;
  return pl;
}

static size_t carve2d(const tsa2d_problem *p, char *base, double **wlut, double **ipow, double **lnn,
                      double **rcp, int32_t **tlab, int32_t **status) {
  Carve c{base};
  const size_t n1 = (size_t)(p->nx * p->ny) + 1;
  *wlut = c.take<double>(n1);
  if (p->q == 1.0) {
    *ipow = nullptr;
    *lnn = c.take<double>(n1);
    *rcp = nullptr;  // S = ln n - W / n: no reciprocal table
  } else {
    *ipow = c.take<double>(n1);
    *lnn = *rcp = nullptr;
  }
  *tlab = c.take<int32_t>((size_t)p->nz);
  *status = c.take<int32_t>((size_t)p->nz);
  return c.off;
}

template <int MODE>
static tsa_status launch2d_mode(const tsa::Tsa2dArgs &a, const Plan2d &pl, cudaStream_t s, bool check) {
  // 256 levels (u8, no overflow possible): the compile-time-L kernel
  auto f = a.L == 256 ? (a.vec ? tsa::k_tsallis2d<MODE, true, false, 256> : tsa::k_tsallis2d<MODE, false, false, 256>)
           : a.vec ? (check ? tsa::k_tsallis2d<MODE, true, true, 0> : tsa::k_tsallis2d<MODE, true, false, 0>)
                   : (check ? tsa::k_tsallis2d<MODE, false, true, 0> : tsa::k_tsallis2d<MODE, false, false, 0>);
  TSA_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)pl.CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.nz * pl.CL));
  cfg.blockDim = dim3(tsa::k2dThreads);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TSA_CUDA(cudaLaunchKernelEx(&cfg, f, a));
  return check_cuda("k_tsallis2d");
}

extern "C" {

tsa_status tsa2d_validate(const tsa2d_problem *p) {
  if (!valid2d(p)) return set_error(TSA_ERR_INVALID_ARG, "2-D problem: volume/dims/bins/q/cluster out of range");
  return TSA_OK;
}

int32_t tsa2d_cluster_size(const tsa2d_problem *p) { return valid2d(p) ? plan2d(p).CL : 0; }

size_t tsa2d_workspace_size(const tsa2d_problem *p) {
  if (!valid2d(p)) return 0;
  double *a, *b, *c, *d;
  int32_t *e, *f;
  return carve2d(p, nullptr, &a, &b, &c, &d, &e, &f);
}

static tsa_status run2d(const tsa2d_problem *p, const tsa_outputs *out, uint32_t *hist_only_out,
                        int32_t *status_only_out, void *workspace, size_t workspace_bytes,
                        cudaStream_t s) {
  double *wlut, *ipow, *lnn, *rcp;
  int32_t *tlab, *status;
  const size_t need = carve2d(p, reinterpret_cast<char *>(workspace), &wlut, &ipow, &lnn, &rcp, &tlab, &status);
  if (!workspace) return set_error(TSA_ERR_INVALID_ARG, "workspace NULL");
  if (workspace_bytes < need) return set_error(TSA_ERR_WORKSPACE, "2-D workspace too small");
  const Plan2d pl = plan2d(p);
  if (pl.smem > kSmem2dMax) return set_error(TSA_ERR_INVALID_ARG, "2-D plan does not fit shared memory (raise cluster)");
  const int64_t N = p->nx * p->ny;
  const bool shannon = p->q == 1.0;
  const bool hist_only = hist_only_out != nullptr;
  if (!hist_only) {
    const int64_t blocks = std::min<int64_t>((N + 256) / 256, 4 * g_num_sms());
    tsa::k2d_luts<<<(unsigned)blocks, 256, 0, s>>>(wlut, ipow, lnn, rcp, N, p->q, shannon);
    TSA_TRY(check_cuda("k2d_luts"));
  }
  tsa::Tsa2dArgs a;
  a.vol = reinterpret_cast<const uint8_t *>(p->volume);
  a.nx = p->nx;
  a.ny = p->ny;
  a.nz = p->nz;
  a.L = p->bins;
  a.LP = pl.LP;
  a.CL = pl.CL;
  a.R = pl.R;
  a.rr = pl.rr;
  a.rounds = pl.rounds;
  a.vec = p->nx % 16 == 0 && (reinterpret_cast<uintptr_t>(p->volume) & 15) == 0;
  a.q = p->q;
  a.mode = shannon ? tsa::SUM : (p->q < 1.0 ? tsa::PROD_MAX : tsa::PROD_MIN);
  a.wlut = wlut;
  a.ipow = ipow;
  a.lnn = lnn;
  a.rcp = rcp;
  a.thresholds = hist_only ? nullptr : out->thresholds;
  a.tlab = hist_only ? nullptr : tlab;
  a.objective = hist_only ? nullptr : out->objective;
  a.hist = hist_only ? hist_only_out : out->histogram;
  a.status = status;
  a.status2 = hist_only ? status_only_out : out->slice_status;
  a.hist_only = hist_only;
  const bool check = p->bins < 256;
  switch (a.mode) {
    case tsa::PROD_MAX: TSA_TRY(launch2d_mode<tsa::PROD_MAX>(a, pl, s, check)); break;
    case tsa::PROD_MIN: TSA_TRY(launch2d_mode<tsa::PROD_MIN>(a, pl, s, check)); break;
    default: TSA_TRY(launch2d_mode<tsa::SUM>(a, pl, s, check)); break;
  }
  if (!hist_only && out->labels) {
    tsa_problem lp = {};
    lp.volume = p->volume;
    lp.dtype = TSA_U8;
    lp.nx = p->nx;
    lp.ny = p->ny;
    lp.nz = p->nz;
    lp.bins = p->bins;
    lp.k = 1;
    lp.q = 1.0;
    TSA_TRY(tsa_label(&lp, tlab, status, out->labels, s));
  }
  return TSA_OK;
}

tsa_status tsa2d_segment(const tsa2d_problem *p, const tsa_outputs *out, void *workspace,
                         size_t workspace_bytes, void *stream) {
  TSA_TRY(tsa2d_validate(p));
  if (!out || !out->thresholds) return set_error(TSA_ERR_INVALID_ARG, "outputs->thresholds NULL");
  return run2d(p, out, nullptr, nullptr, workspace, workspace_bytes, S(stream));
}

tsa_status tsa2d_histogram(const tsa2d_problem *p, uint32_t *hist, int32_t *slice_status,
                           void *workspace, size_t workspace_bytes, void *stream) {
  TSA_TRY(tsa2d_validate(p));
  if (!hist || !slice_status) return set_error(TSA_ERR_INVALID_ARG, "hist/slice_status NULL");
  return run2d(p, nullptr, hist, slice_status, workspace, workspace_bytes, S(stream));
}

tsa_status tsa2d_mean3x3(const tsa2d_problem *p, uint8_t *g, void *stream) {
  TSA_TRY(tsa2d_validate(p));
  if (!g) return set_error(TSA_ERR_INVALID_ARG, "g NULL");
  const int vec = p->nx % 4 == 0 && (reinterpret_cast<uintptr_t>(p->volume) & 3) == 0 &&
                  (reinterpret_cast<uintptr_t>(g) & 3) == 0;
  const int64_t items = vec ? p->nx / 4 * p->ny : p->nx * p->ny;
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(64, (items + 255) / 256));
  tsa::k2d_mean<<<dim3(gx, (unsigned)p->nz), 256, 0, S(stream)>>>(
      reinterpret_cast<const uint8_t *>(p->volume), g, p->nx, p->ny, vec);
  return check_cuda("k2d_mean");
}

// ------------------------------------------------------------- HU input
static bool valid_hu(const tsa_hu_problem *p) {
  if (!p || !p->volume || p->nx <= 0 || p->ny <= 0 || p->nz <= 0 || p->nz > 65535) return false;
  const int64_t n = p->nx * p->ny;
  if (n >= (int64_t(1) << 31) || n % 16 != 0) return false;
  if ((reinterpret_cast<uintptr_t>(p->volume) & 15) != 0) return false;
  if (p->background < -tsa::kHuOff || p->background >= tsa::kHuBins - tsa::kHuOff) return false;
  return valid_search_shape(p->nz, n, 256, p->k, p->q, p->objective, p->enumeration);
}

struct HuWs {
  uint32_t *hu_hist, *hist8;
  uint8_t *glut;
  int32_t *win, *status;
  double *ps;
  uint64_t *pk;
  char *search;
  size_t search_bytes;
  int32_t units;
  double *luts;  // small class-term table (Luts::sp) for the per-slice search kernel
};

static size_t carve_hu(const tsa_hu_problem *p, char *base, HuWs *o) {
  Carve c{base};
  HuWs w;
  const int64_t n = p->nx * p->ny;
  w.units = tsa_default_units(p->nz, 256, p->k, p->enumeration);
  w.hu_hist = c.take<uint32_t>((size_t)p->nz * tsa::kHuBins);
  w.hist8 = c.take<uint32_t>((size_t)p->nz * 256);
  w.glut = c.take<uint8_t>(tsa::kHuBins);
  w.win = c.take<int32_t>(4);
  w.status = c.take<int32_t>((size_t)p->nz);
  w.ps = c.take<double>((size_t)w.units * p->nz);
  w.pk = c.take<uint64_t>((size_t)w.units * p->nz);
  w.search_bytes = tsa_search_workspace_size(p->nz, n, 256, p->k, p->q, p->objective, p->enumeration);
  w.search = c.take<char>(w.search_bytes);
  w.luts = c.take<double>(tsa::kSmallLut);
  if (o) *o = w;
  return c.off;
}

size_t tsa_hu_workspace_size(const tsa_hu_problem *p) {
  if (!valid_hu(p)) return 0;
  return carve_hu(p, nullptr, nullptr);
}

static tsa_status hu_window_pass(const tsa_hu_problem *p, const HuWs &w, cudaStream_t s) {
  const int64_t n = p->nx * p->ny;
  TSA_CUDA(cudaMemsetAsync(w.hu_hist, 0, sizeof(uint32_t) * p->nz * tsa::kHuBins, s));
  TSA_CUDA(cudaMemsetAsync(w.status, 0, sizeof(int32_t) * p->nz, s));
  tsa::k_hu_init<<<1, 1, 0, s>>>(w.win);
  tsa::HuArgs a;
  a.vol = p->volume;
  a.n = n;
  a.nz = p->nz;
  a.bg = p->background;
  a.hu_hist = w.hu_hist;
  a.win = w.win;
  a.status = w.status;
  // <= 128 K voxels per CTA (a 16-bit counter copy serves 4 of 16 warps:
  // < 32 K counts); 64 KB of bins: three CTAs per SM
  a.chunks = (int)std::max<int64_t>(1, std::min<int64_t>(4096, (n + 131071) / 131072));
  const size_t smem = (size_t)4 * (tsa::kHuBins / 2) * sizeof(uint32_t);
  TSA_CUDA(cudaFuncSetAttribute(tsa::k_hu_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  tsa::k_hu_hist<<<dim3((unsigned)a.chunks, (unsigned)p->nz), 512, smem, s>>>(a);
  TSA_TRY(check_cuda("k_hu_hist"));
  tsa::k_hu_window<<<dim3(tsa::kHuBins / 256, (unsigned)std::min<int64_t>(p->nz, 16)), 256, 0, s>>>(
      w.hu_hist, p->nz, p->background, w.win);
  tsa::k_hu_window_fold<<<1, 1, 0, s>>>(w.win);
  return check_cuda("k_hu_window");
}

static tsa_status hu_finish_impl(const tsa_hu_problem *p, const int32_t *win, const tsa_outputs *out,
                                 const HuWs &w, void *stream) {
  cudaStream_t s = S(stream);
  const int64_t n = p->nx * p->ny;
  uint32_t *hist8 = out->histogram ? out->histogram : w.hist8;
  TSA_CUDA(cudaMemsetAsync(hist8, 0, sizeof(uint32_t) * p->nz * 256, s));
  tsa::k_hu_glut<<<tsa::kHuBins / 256, 256, 0, s>>>(win, p->background, w.glut);
  tsa::k_hu_remap<<<dim3(4, (unsigned)p->nz), 256, 0, s>>>(w.hu_hist, w.glut, hist8);
  TSA_TRY(check_cuda("k_hu_remap"));
  if (p->k <= 2 && p->enumeration == TSA_ENUM_CANONICAL && p->objective == TSA_OBJ_PSEUDO_ADDITIVE) {
    // the compact path's per-slice kernel (tables, canonical search, argmax,
    // phi(t*) in the definition's order; one CTA per slice) on the remapped
    // histograms: one partial per slice, the overflow flag = the HU status
    const bool shannon = p->q == 1.0;
    tsa::FusedArgs a = {};
    a.n = n;
    a.nz = p->nz;
    a.L = 256;
    a.k = p->k;
    a.q = p->q;
    a.mode = search_mode(p->q, p->objective);
    a.thresholds = out->thresholds;
    a.objective = out->objective;
    a.hist = hist8;
    a.status = w.status;
    a.status2 = out->slice_status;
    a.partial = hist8;
    a.povf = w.status;
    a.counters = nullptr;
    (void)shannon;
    a.sp = w.luts;
    a.luts = make_luts(p->q, w.luts);
    a.HC = 1;
    const int lgrid = (tsa::kSmallLut + 255) / 256;
    tsa::k_lut_part<<<lgrid, 256, 0, s>>>(a);
    TSA_TRY(check_cuda("k_lut_part"));
    const int L = 256, E = L + 1;
    const size_t sm = (size_t)((L + 1) & ~1) * 4 + (size_t)L * 8 * 3 + (size_t)E * 8 * 2 + (size_t)E * 8 + 64;
    auto mid = p->k == 1 ? (a.mode == tsa::PROD_MAX ? tsa::k_mid<1, tsa::PROD_MAX>
                            : a.mode == tsa::PROD_MIN ? tsa::k_mid<1, tsa::PROD_MIN> : tsa::k_mid<1, tsa::SUM>)
                         : (a.mode == tsa::PROD_MAX ? tsa::k_mid<2, tsa::PROD_MAX>
                            : a.mode == tsa::PROD_MIN ? tsa::k_mid<2, tsa::PROD_MIN> : tsa::k_mid<2, tsa::SUM>);
    if (sm > 48 * 1024) cudaFuncSetAttribute(mid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    mid<<<(unsigned)p->nz, tsa::kMidThreads, sm, s>>>(a);
    TSA_TRY(check_cuda("k_mid (HU)"));
  } else {
    TSA_TRY(tsa_search(hist8, w.status, p->nz, n, 256, p->k, p->q, p->objective, p->enumeration, w.units, 0,
                       w.units, w.ps, w.pk, w.search, w.search_bytes, stream));
    TSA_TRY(finalize_impl(hist8, w.status, p->nz, 256, p->k, p->q, p->objective, w.ps, w.pk, w.units,
                          out->thresholds, out->objective, w.status, out->slice_status, s));
  }
  if (out->labels) {
    const dim3 grid(4, (unsigned)p->nz);  // 4 contiguous chunks per slice
    switch (p->k) {
      case 1: tsa::k_label_hu<1><<<grid, 256, 0, s>>>(p->volume, out->labels, out->thresholds, w.status, win, p->background, n, p->k); break;
      case 2: tsa::k_label_hu<2><<<grid, 256, 0, s>>>(p->volume, out->labels, out->thresholds, w.status, win, p->background, n, p->k); break;
      case 3: tsa::k_label_hu<3><<<grid, 256, 0, s>>>(p->volume, out->labels, out->thresholds, w.status, win, p->background, n, p->k); break;
      default: tsa::k_label_hu<4><<<grid, 256, 0, s>>>(p->volume, out->labels, out->thresholds, w.status, win, p->background, n, p->k); break;
    }
    TSA_TRY(check_cuda("k_label_hu"));
  }
  return TSA_OK;
}

static tsa_status hu_check(const tsa_hu_problem *p, const tsa_outputs *out, void *workspace,
                           size_t workspace_bytes, HuWs *w) {
  if (!valid_hu(p)) return set_error(TSA_ERR_INVALID_ARG, "HU problem: dims/alignment/k/q/objective");
  if (out && !out->thresholds) return set_error(TSA_ERR_INVALID_ARG, "outputs->thresholds NULL");
  if (out && out->labels && (reinterpret_cast<uintptr_t>(out->labels) & 15) != 0)
    return set_error(TSA_ERR_INVALID_ARG, "labels not 16-byte aligned");
  if (!workspace) return set_error(TSA_ERR_INVALID_ARG, "workspace NULL");
  const size_t need = carve_hu(p, reinterpret_cast<char *>(workspace), w);
  if (workspace_bytes < need) return set_error(TSA_ERR_WORKSPACE, "HU workspace too small");
  return TSA_OK;
}

tsa_status tsa_hu_segment(const tsa_hu_problem *p, const tsa_outputs *out, int32_t *window,
                          void *workspace, size_t workspace_bytes, void *stream) {
  if (!out) return set_error(TSA_ERR_INVALID_ARG, "outputs NULL");
  HuWs w;
  TSA_TRY(hu_check(p, out, workspace, workspace_bytes, &w));
  cudaStream_t s = S(stream);
  TSA_TRY(hu_window_pass(p, w, s));
  TSA_TRY(hu_finish_impl(p, w.win, out, w, stream));
  if (window) TSA_CUDA(cudaMemcpyAsync(window, w.win, 2 * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  return TSA_OK;
}

tsa_status tsa_hu_histogram(const tsa_hu_problem *p, int32_t *window_out, void *workspace,
                            size_t workspace_bytes, void *stream) {
  if (!window_out) return set_error(TSA_ERR_INVALID_ARG, "window_out NULL");
  HuWs w;
  TSA_TRY(hu_check(p, nullptr, workspace, workspace_bytes, &w));
  cudaStream_t s = S(stream);
  TSA_TRY(hu_window_pass(p, w, s));
  TSA_CUDA(cudaMemcpyAsync(window_out, w.win, 2 * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  return TSA_OK;
}

tsa_status tsa_hu_finish(const tsa_hu_problem *p, const int32_t *window_in, const tsa_outputs *out,
                         void *workspace, size_t workspace_bytes, void *stream) {
  if (!out || !window_in) return set_error(TSA_ERR_INVALID_ARG, "outputs/window_in NULL");
  HuWs w;
  TSA_TRY(hu_check(p, out, workspace, workspace_bytes, &w));
  return hu_finish_impl(p, window_in, out, w, stream);
}

tsa_status tsa_hu_preprocess(const tsa_hu_problem *p, uint8_t *gray, int32_t *window, void *workspace,
                             size_t workspace_bytes, void *stream) {
  if (!valid_hu(p)) return set_error(TSA_ERR_INVALID_ARG, "HU problem: dims/alignment/k/q/objective");
  if (!gray || !workspace) return set_error(TSA_ERR_INVALID_ARG, "gray/workspace NULL");
  HuWs w;
  const size_t need = carve_hu(p, reinterpret_cast<char *>(workspace), &w);
  if (workspace_bytes < need) return set_error(TSA_ERR_WORKSPACE, "HU workspace too small");
  cudaStream_t s = S(stream);
  TSA_TRY(hu_window_pass(p, w, s));
  const int64_t total = p->nx * p->ny * p->nz;
  const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)g_num_sms() * 8);
  tsa::k_hu_map<<<blocks, 256, 0, s>>>(p->volume, gray, w.win, p->background, total);
  TSA_TRY(check_cuda("k_hu_map"));
  if (window) TSA_CUDA(cudaMemcpyAsync(window, w.win, 2 * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  return TSA_OK;
}

// ------------------------------------------------------------ morphology
}  // extern "C"

template <int R, bool MAX, bool TOPHAT>
static tsa_status launch_morph_r(const tsa::MorphArgs &a, cudaStream_t s) {
  const dim3 grid((unsigned)((a.nx + tsa::kMorphStrip - 1) / tsa::kMorphStrip),
                  (unsigned)((a.ny + tsa::kMorphChunk - 1) / tsa::kMorphChunk), (unsigned)a.nz);
  tsa::k_morph<R, MAX, TOPHAT><<<grid, tsa::kMorphThreads, 0, s>>>(a);
  return check_cuda("k_morph");
}

template <bool MAX, bool TOPHAT>
static tsa_status launch_morph(int r, const tsa::MorphArgs &a, cudaStream_t s) {
  switch (r) {
    case 1: return launch_morph_r<1, MAX, TOPHAT>(a, s);
    case 2: return launch_morph_r<2, MAX, TOPHAT>(a, s);
    case 3: return launch_morph_r<3, MAX, TOPHAT>(a, s);
    case 4: return launch_morph_r<4, MAX, TOPHAT>(a, s);
    case 5: return launch_morph_r<5, MAX, TOPHAT>(a, s);
    case 6: return launch_morph_r<6, MAX, TOPHAT>(a, s);
    case 7: return launch_morph_r<7, MAX, TOPHAT>(a, s);
    case 8: return launch_morph_r<8, MAX, TOPHAT>(a, s);
    case 9: return launch_morph_r<9, MAX, TOPHAT>(a, s);
    default: return launch_morph_r<10, MAX, TOPHAT>(a, s);
  }
}

extern "C" {

size_t tsa_morph_workspace_size(int64_t nx, int64_t ny, int64_t nz, int32_t op) {
  if (nx <= 0 || ny <= 0 || nz <= 0) return 0;
  return (op == TSA_MORPH_OPEN || op == TSA_MORPH_TOPHAT) ? align_up((size_t)(nx * ny * nz)) : 0;
}

tsa_status tsa_morph(const uint8_t *in, uint8_t *out, int64_t nx, int64_t ny, int64_t nz,
                     int32_t radius, int32_t op, void *workspace, size_t workspace_bytes,
                     void *stream) {
  if (!in || !out || in == out || nx <= 0 || ny <= 0 || nz <= 0 || nz > 65535 || nx * ny >= (int64_t(1) << 31) ||
      radius < 0 || radius > tsa::kMorphRmax || op < TSA_MORPH_ERODE || op > TSA_MORPH_TOPHAT)
    return set_error(TSA_ERR_INVALID_ARG, "morph: pointers/dims/radius (0..10)/op");
  cudaStream_t s = S(stream);
  const size_t vb = (size_t)(nx * ny * nz);
  const bool two = op == TSA_MORPH_OPEN || op == TSA_MORPH_TOPHAT;
  if (two && (!workspace || workspace_bytes < vb)) return set_error(TSA_ERR_WORKSPACE, "morph workspace");
  if (radius == 0) {  // disk(0) = the origin: erosion / dilation / opening are the identity
    if (op == TSA_MORPH_TOPHAT) TSA_CUDA(cudaMemsetAsync(out, 0, vb, s));
    else TSA_CUDA(cudaMemcpyAsync(out, in, vb, cudaMemcpyDeviceToDevice, s));
    return TSA_OK;
  }
  tsa::MorphArgs a;
  a.nx = nx;
  a.ny = ny;
  a.nz = nz;
  a.orig = nullptr;
  if (op == TSA_MORPH_ERODE || op == TSA_MORPH_DILATE) {
    a.src = in;
    a.dst = out;
    return op == TSA_MORPH_ERODE ? launch_morph<false, false>(radius, a, s) : launch_morph<true, false>(radius, a, s);
  }
  uint8_t *e = reinterpret_cast<uint8_t *>(workspace);
  a.src = in;
  a.dst = e;
  TSA_TRY((launch_morph<false, false>(radius, a, s)));
  a.src = e;
  a.dst = out;
  if (op == TSA_MORPH_OPEN) return launch_morph<true, false>(radius, a, s);
  a.orig = in;
  return launch_morph<true, true>(radius, a, s);
}

// ----------------------------------------------------------- host buffers
static size_t slab_bytes(const tsa_problem *p, int64_t slab, tsa_problem *sp) {
  *sp = *p;
  sp->nz = slab;
  sp->volume = reinterpret_cast<const void *>(uintptr_t(1));  // shape only
  const size_t vb = (size_t)slab * p->nx * p->ny * (p->dtype == TSA_U8 ? 1 : 2);
  const size_t lb = (size_t)slab * p->nx * p->ny;
  Carve c{nullptr};
  c.take<char>(vb);
  c.take<char>(lb);
  c.take<char>(tsa_workspace_size(sp));
  return c.off;
}

// per-volume device arrays of the small outputs (copied to the host once)
static size_t small_bytes(const tsa_problem *p) {
  Carve c{nullptr};
  c.take<int32_t>((size_t)p->nz * p->k);
  c.take<double>((size_t)p->nz);
  c.take<int32_t>((size_t)p->nz);
  return c.off;
}

// device slab buffers of tsa_segment_host: with two, the copy-in of slab i+2
// waited for slab i's labels to leave, i.e. for slab i's compute -- a bubble
// of one compute latency per slab on the H2D engine; three keep both copy
// engines streaming
constexpr int kHostBufs = 3;

size_t tsa_segment_host_scratch_size(const tsa_problem *p, int64_t slab) {
  if (tsa_validate(p) != TSA_OK || slab <= 0) return 0;
  slab = std::min(slab, p->nz);
  tsa_problem sp;
  return (size_t)kHostBufs * slab_bytes(p, slab, &sp) + small_bytes(p);
}

tsa_status tsa_segment_host(const tsa_problem *p, int64_t slab, int32_t *thr_h, double *obj_h,
                            int32_t *st_h, uint8_t *lab_h, void *dev_buf, size_t dev_bytes,
                            void *stream0, void *stream1) {
  TSA_TRY(tsa_validate(p));
  if (slab <= 0 || !thr_h || !dev_buf) return set_error(TSA_ERR_INVALID_ARG, "host segment args");
  slab = std::min(slab, p->nz);
  tsa_problem sp;
  const size_t per = slab_bytes(p, slab, &sp);
  if (dev_bytes < kHostBufs * per + small_bytes(p)) return set_error(TSA_ERR_WORKSPACE, "device scratch too small");
  const size_t esz = p->dtype == TSA_U8 ? 1 : 2;
  const int64_t n = p->nx * p->ny;
  Carve cs{reinterpret_cast<char *>(dev_buf) + kHostBufs * per};
  int32_t *thr_all = cs.take<int32_t>((size_t)p->nz * p->k);
  double *obj_all = cs.take<double>((size_t)p->nz);
  int32_t *sts_all = cs.take<int32_t>((size_t)p->nz);
  // Three streams: copy-in on a stream of this call (created and destroyed
  // here: the call blocks anyway), compute on stream0, copy-out on stream1.
  // kHostBufs device buffers: slab i+3 may overwrite buffer i%3 once slab i's
  // labels left (ev_free); slab i is computed once it arrived (ev_in) and its labels
  // leave once it is computed (ev_done) -- so the H2D engine streams slab i+1
  // while the kernels run on slab i and the D2H engine drains slab i-1.
  // Thresholds, objective and status stay on the device for the whole volume
  // and are copied once at the end.
  cudaStream_t comp = S(stream0), cout = S(stream1), cin = comp;
  // one slab: nothing to overlap the copy-in with (and no stream to create:
  // c1's single 256^2 slice is latency-bound)
  const bool own_in = p->nz > slab;
  if (own_in) TSA_CUDA(cudaStreamCreateWithFlags(&cin, cudaStreamNonBlocking));
  cudaEvent_t ev_done[kHostBufs], ev_free[kHostBufs], ev_in[kHostBufs], ev_start;
  for (int b = 0; b < kHostBufs; b++) {
    TSA_CUDA(cudaEventCreateWithFlags(&ev_done[b], cudaEventDisableTiming));
    TSA_CUDA(cudaEventCreateWithFlags(&ev_free[b], cudaEventDisableTiming));
    TSA_CUDA(cudaEventCreateWithFlags(&ev_in[b], cudaEventDisableTiming));
  }
  TSA_CUDA(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
  // the copy-in stream starts after work already queued on stream0
  TSA_CUDA(cudaEventRecord(ev_start, comp));
  TSA_CUDA(cudaStreamWaitEvent(cin, ev_start, 0));
  tsa_status rc = TSA_OK;
  for (int64_t z0 = 0, i = 0; z0 < p->nz && rc == TSA_OK; z0 += slab, i++) {
    const int64_t nzs = std::min(slab, p->nz - z0);
    const int b = (int)(i % kHostBufs);
    Carve c{reinterpret_cast<char *>(dev_buf) + b * per};
    char *vol = c.take<char>((size_t)slab * n * esz);
    uint8_t *lab = c.take<uint8_t>((size_t)slab * n);
    int32_t *thr = thr_all + z0 * p->k;
    double *obj = obj_all + z0;
    int32_t *sts = sts_all + z0;
    tsa_problem q = *p;
    q.nz = nzs;
    q.volume = vol;
    char *ws = c.take<char>(0);
    const size_t wsb = tsa_workspace_size(&q);
    const char *src = reinterpret_cast<const char *>(p->volume) + (size_t)z0 * n * esz;
    if (i >= kHostBufs && cudaStreamWaitEvent(cin, ev_free[b], 0) != cudaSuccess)
      rc = set_error(TSA_ERR_CUDA, "wait ev_free");
    if (rc == TSA_OK && cudaMemcpyAsync(vol, src, (size_t)nzs * n * esz, cudaMemcpyHostToDevice, cin) != cudaSuccess)
      rc = set_error(TSA_ERR_CUDA, "H2D");
    if (rc == TSA_OK && (cudaEventRecord(ev_in[b], cin) != cudaSuccess ||
                         cudaStreamWaitEvent(comp, ev_in[b], 0) != cudaSuccess))
      rc = set_error(TSA_ERR_CUDA, "ev_in");
    // the compute of slab i reuses the workspace of buffer b: ordered after
    // slab i-2's compute by stream order on comp
    tsa_outputs o{thr, lab_h ? lab : nullptr, obj, nullptr, sts};
    if (rc == TSA_OK) rc = tsa_segment(&q, &o, ws, wsb, comp);
    if (rc != TSA_OK) break;
    if (!lab_h && cudaEventRecord(ev_free[b], comp) != cudaSuccess) rc = set_error(TSA_ERR_CUDA, "ev_free");
    if (lab_h) {
      cudaError_t e = cudaEventRecord(ev_done[b], comp);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(cout, ev_done[b], 0);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(lab_h + (size_t)z0 * n, lab, (size_t)nzs * n, cudaMemcpyDeviceToHost, cout);
      if (e == cudaSuccess) e = cudaEventRecord(ev_free[b], cout);
      if (e != cudaSuccess) rc = set_error(TSA_ERR_CUDA, "D2H labels");
    }
  }
  if (rc == TSA_OK) {
    cudaError_t e = cudaMemcpyAsync(thr_h, thr_all, sizeof(int32_t) * p->nz * p->k, cudaMemcpyDeviceToHost, comp);
    if (e == cudaSuccess && obj_h)
      e = cudaMemcpyAsync(obj_h, obj_all, sizeof(double) * p->nz, cudaMemcpyDeviceToHost, comp);
    if (e == cudaSuccess && st_h)
      e = cudaMemcpyAsync(st_h, sts_all, sizeof(int32_t) * p->nz, cudaMemcpyDeviceToHost, comp);
    if (e != cudaSuccess) rc = set_error(TSA_ERR_CUDA, "D2H results");
  }
  const cudaError_t e0 = cudaStreamSynchronize(comp), e1 = cudaStreamSynchronize(cout),
                    e2 = own_in ? cudaStreamSynchronize(cin) : cudaSuccess;
  for (int b = 0; b < kHostBufs; b++) {
    cudaEventDestroy(ev_done[b]);
    cudaEventDestroy(ev_free[b]);
    cudaEventDestroy(ev_in[b]);
  }
  cudaEventDestroy(ev_start);
  if (own_in) cudaStreamDestroy(cin);
  if (rc != TSA_OK) return rc;
  if (e0 != cudaSuccess || e1 != cudaSuccess || e2 != cudaSuccess)
    return set_error(TSA_ERR_CUDA, "tsa_segment_host synchronize");
  return TSA_OK;
}

#ifdef TSA_TRACE
// debug builds only (tools/fused_trace.py): copy the fused-kernel task trace to the host
int tsa_debug_trace(unsigned long long *host, int max_entries) {
  int n = 0;
  cudaMemcpyFromSymbol(&n, tsa::g_trace_n, sizeof(int));
  n = std::min(n, std::min(max_entries, 65536));
  cudaMemcpyFromSymbol(host, tsa::g_trace, sizeof(unsigned long long) * 5 * n);
  const int zero = 0;
  cudaMemcpyToSymbol(tsa::g_trace_n, &zero, sizeof(int));
  return n;
}
int tsa_debug_sphase(unsigned long long *host, int nz) {
  cudaMemcpyFromSymbol(host, tsa::g_sphase, sizeof(unsigned long long) * 8 * std::min(nz, 4096));
  return 0;
}
int tsa_debug_mphase(unsigned long long *host, int nz) {
  cudaMemcpyFromSymbol(host, tsa::g_mphase, sizeof(unsigned long long) * 8 * std::min(nz, 4096));
  return 0;
}
#endif
}  // extern "C"
