// tsa_comm.cu -- multi-GPU entry points of libtsa (include/tsa.h, "multi-GPU"):
// the all-gather transport (NCCL, loaded with dlopen, or a caller-provided
// all-gather) and tsa_segment_sharded, which sequences the C-ABI stage calls
// around the two exchanges of the tuple-sharded path (
// PAPER.md:724 "job distribution ... reduction of results from different
// devices").  Every step of the path runs in the libtsa kernels; this file
// only orders them and moves the histograms and (score, key) partials.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types and enum values only; the functions come from dlsym

#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "tsa.h"
#include "tsa_internal.h"

struct tsa_comm {
  int32_t nranks = 0, rank = 0, kind = 0;  // kind: 1 NCCL, 2 custom
  ncclComm_t nc = nullptr;
  tsa_allgather_fn fn = nullptr;
  void *user = nullptr;
};

namespace {

constexpr int kNccl = 1, kCustom = 2;
// Work units per slice of the sharded search are computed for this SM count
// on every rank (B200), never the local device's, so all ranks agree.
constexpr int32_t kShardRefSms = 148;

tsa_status fail(tsa_status s, const std::string &msg) {
  tsa_internal_set_error(msg.c_str());
  return s;
}

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

// libnccl.so.2 is resolved at the first NCCL call (in a PyTorch process the
// copy torch already mapped is returned); nothing links libtsa to NCCL.
NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("dlopen libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char *n) { return dlsym(h, n); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.GroupStart &&
             api.GroupEnd && api.GetErrorString;
    if (!api.ok) api.err = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

tsa_status nccl_check(ncclResult_t r, const char *where) {
  if (r == ncclSuccess) return TSA_OK;
  return fail(TSA_ERR_NCCL, std::string(where) + ": " + nccl().GetErrorString(r));
}

// Rank-major all-gather of `bytes` per rank on `s`.
tsa_status allgather(tsa_comm *c, const void *send, void *recv, size_t bytes, cudaStream_t s) {
  if (c->kind == kNccl)
    return nccl_check(nccl().AllGather(send, recv, bytes, ncclUint8, c->nc, s), "ncclAllGather");
  if (c->fn(c->user, send, recv, bytes, reinterpret_cast<void *>(s)) != 0)
    return fail(TSA_ERR_NCCL, "custom all-gather returned an error");
  return TSA_OK;
}

// (-inf, TSA_KEY_NONE): "no tuple" partials of a rank without work units
__global__ void k_fill_none(double *score, uint64_t *key, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    score[i] = -INFINITY;
    key[i] = TSA_KEY_NONE;
  }
}

constexpr size_t kAlign = 256;
struct Carve {
  char *base;
  size_t off = 0;
  template <typename T>
  T *take(size_t count) {
    T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
    off += (count * sizeof(T) + kAlign - 1) / kAlign * kAlign;
    return p;
  }
};

struct ShardWs {
  uint32_t *hist_all;  // [P * per][bins]
  int32_t *st_all;     // [P * per]
  int32_t *st_work;    // [nz_total]
  double *ps;          // [cu][nz_total]
  uint64_t *pk;
  double *ms;          // [P][nz_total]
  uint64_t *mk;
  char *search;
  size_t search_bytes;
};

// A shape-only copy of the slab problem for nz slices (validation / sizes).
tsa_problem shape_of(const tsa_problem *slab, int64_t nz) {
  tsa_problem p = *slab;
  p.nz = nz;
  if (!p.volume) p.volume = reinterpret_cast<const void *>(uintptr_t(256));
  return p;
}

bool comm_ok(const tsa_comm *c) { return c && c->nranks >= 1 && c->rank >= 0 && c->rank < c->nranks; }

int64_t per_rank(int64_t nz_total, int32_t P) { return (nz_total + P - 1) / P; }

size_t carve_shard(const tsa_problem *slab, int64_t nz_total, int32_t P, char *base, ShardWs *o) {
  const int64_t per = per_rank(nz_total, P);
  const int32_t U = tsa_sharded_units(slab, nz_total, P);
  const int64_t cu = std::max<int64_t>(1, (U + P - 1) / P);
  Carve c{base};
  ShardWs w;
  w.hist_all = c.take<uint32_t>((size_t)P * per * slab->bins);
  w.st_all = c.take<int32_t>((size_t)P * per);
  w.st_work = c.take<int32_t>((size_t)nz_total);
  w.ps = c.take<double>((size_t)cu * nz_total);
  w.pk = c.take<uint64_t>((size_t)cu * nz_total);
  w.ms = c.take<double>((size_t)P * nz_total);
  w.mk = c.take<uint64_t>((size_t)P * nz_total);
  w.search_bytes = tsa_search_workspace_size(nz_total, slab->nx * slab->ny, slab->bins, slab->k, slab->q,
                                             slab->objective, slab->enumeration);
  w.search = c.take<char>(w.search_bytes);
  if (o) *o = w;
  return c.off;
}

}  // namespace

extern "C" {

tsa_status tsa_comm_unique_id(unsigned char id[TSA_COMM_ID_BYTES]) {
  if (!id) return fail(TSA_ERR_INVALID_ARG, "id is NULL");
  NcclApi &api = nccl();
  if (!api.ok) return fail(TSA_ERR_NCCL, api.err);
  ncclUniqueId u;
  if (nccl_check(api.GetUniqueId(&u), "ncclGetUniqueId") != TSA_OK) return TSA_ERR_NCCL;
  static_assert(sizeof(u) == TSA_COMM_ID_BYTES, "NCCL unique id size");
  memcpy(id, &u, sizeof(u));
  return TSA_OK;
}

tsa_status tsa_comm_init(tsa_comm **comm, int32_t nranks, int32_t rank, const unsigned char id[TSA_COMM_ID_BYTES]) {
  if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(TSA_ERR_INVALID_ARG, "tsa_comm_init arguments");
  *comm = nullptr;
  NcclApi &api = nccl();
  if (!api.ok) return fail(TSA_ERR_NCCL, api.err);
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  ncclComm_t nc = nullptr;
  if (nccl_check(api.CommInitRank(&nc, nranks, u, rank), "ncclCommInitRank") != TSA_OK) return TSA_ERR_NCCL;
  tsa_comm *c = new (std::nothrow) tsa_comm;
  if (!c) {
    api.CommDestroy(nc);
    return fail(TSA_ERR_INVALID_ARG, "out of host memory");
  }
  c->nranks = nranks;
  c->rank = rank;
  c->kind = kNccl;
  c->nc = nc;
  *comm = c;
  return TSA_OK;
}

tsa_status tsa_comm_init_custom(tsa_comm **comm, int32_t nranks, int32_t rank, tsa_allgather_fn fn, void *user) {
  if (!comm || !fn || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(TSA_ERR_INVALID_ARG, "tsa_comm_init_custom arguments");
  tsa_comm *c = new (std::nothrow) tsa_comm;
  if (!c) return fail(TSA_ERR_INVALID_ARG, "out of host memory");
  c->nranks = nranks;
  c->rank = rank;
  c->kind = kCustom;
  c->fn = fn;
  c->user = user;
  *comm = c;
  return TSA_OK;
}

tsa_status tsa_comm_destroy(tsa_comm *comm) {
  if (!comm) return TSA_OK;
  tsa_status rc = TSA_OK;
  if (comm->kind == kNccl && comm->nc) rc = nccl_check(nccl().CommDestroy(comm->nc), "ncclCommDestroy");
  delete comm;
  return rc;
}

int32_t tsa_comm_kind(const tsa_comm *comm) { return comm ? comm->kind : 0; }

tsa_status tsa_slab_range(int64_t nz_total, int32_t nranks, int32_t rank, int64_t *z0, int64_t *z1) {
  if (nz_total < 0 || nranks < 1 || rank < 0 || rank >= nranks || !z0 || !z1)
    return fail(TSA_ERR_INVALID_ARG, "tsa_slab_range arguments");
  const int64_t per = per_rank(nz_total, nranks);
  *z0 = std::min(nz_total, (int64_t)rank * per);
  *z1 = std::min(nz_total, *z0 + per);
  return TSA_OK;
}

int32_t tsa_sharded_units(const tsa_problem *slab, int64_t nz_total, int32_t nranks) {
  if (!slab || nz_total <= 0 || nranks < 1) return 0;
  if (slab->enumeration == TSA_ENUM_DP) return 1;  // one unit per slice (tsa_search)
  if (slab->units_per_slice > 0) return slab->units_per_slice;
  const int32_t u = tsa_units_for_sms(nz_total, slab->bins, slab->k, slab->enumeration, kShardRefSms);
  return std::max(u, nranks);
}

size_t tsa_sharded_workspace_size(const tsa_problem *slab, int64_t nz_total, int32_t mode, const tsa_comm *comm) {
  if (!slab || !comm_ok(comm) || nz_total <= 0) return 0;
  if (mode == TSA_SHARD_SLICES) return slab->nz > 0 ? tsa_workspace_size(slab) : 0;
  if (mode != TSA_SHARD_TUPLES) return 0;
  const tsa_problem shape = shape_of(slab, nz_total);
  if (tsa_validate(&shape) != TSA_OK) return 0;
  return carve_shard(&shape, nz_total, comm->nranks, nullptr, nullptr);
}

tsa_status tsa_segment_sharded(const tsa_problem *slab, int64_t nz_total, const tsa_outputs *out, int32_t mode,
                               tsa_comm *comm, void *workspace, size_t workspace_bytes, void *stream) {
  if (!slab || !out || !comm_ok(comm)) return fail(TSA_ERR_INVALID_ARG, "sharded: slab / outputs / comm");
  int64_t z0, z1;
  if (tsa_slab_range(nz_total, comm->nranks, comm->rank, &z0, &z1) != TSA_OK)
    return fail(TSA_ERR_INVALID_ARG, "sharded: nz_total");
  if (slab->nz != z1 - z0) return fail(TSA_ERR_INVALID_ARG, "sharded: slab->nz != the rank's tsa_slab_range");
  if (mode == TSA_SHARD_SLICES) {
    if (slab->nz == 0) return TSA_OK;
    return tsa_segment(slab, out, workspace, workspace_bytes, stream);
  }
  if (mode != TSA_SHARD_TUPLES) return fail(TSA_ERR_INVALID_ARG, "sharded: shard_mode");
  const tsa_problem shape = shape_of(slab, nz_total);
  if (tsa_validate(&shape) != TSA_OK) return TSA_ERR_INVALID_ARG;  // detail set by tsa_validate
  if (slab->nz > 0 && !slab->volume) return fail(TSA_ERR_INVALID_ARG, "sharded: volume NULL");
  if (!out->thresholds) return fail(TSA_ERR_INVALID_ARG, "sharded: outputs->thresholds NULL");
  if (!workspace) return fail(TSA_ERR_INVALID_ARG, "sharded: workspace NULL");
  const int32_t P = comm->nranks, r = comm->rank;
  ShardWs w;
  if (workspace_bytes < carve_shard(&shape, nz_total, P, reinterpret_cast<char *>(workspace), &w))
    return fail(TSA_ERR_WORKSPACE, "sharded workspace too small");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int64_t per = per_rank(nz_total, P);
  const int32_t L = slab->bins, k = slab->k;
  auto cuda = [&](cudaError_t e, const char *where) -> tsa_status {
    if (e == cudaSuccess) return TSA_OK;
    return fail(TSA_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
  };
#define SH_TRY(x)                  \
  do {                             \
    tsa_status _s = (x);           \
    if (_s != TSA_OK) return _s;   \
  } while (0)
  // 1. histogram of the own slab into the rank's block (in-place all-gather)
  uint32_t *hown = w.hist_all + (size_t)r * per * L;
  int32_t *sown = w.st_all + (size_t)r * per;
  if (slab->nz > 0) SH_TRY(tsa_histogram(slab, hown, sown, stream));
  // 2. every rank gets every slice's histogram and status (rows >= nz_total unused)
  if (comm->kind == kNccl) SH_TRY(nccl_check(nccl().GroupStart(), "ncclGroupStart"));
  tsa_status rc = allgather(comm, hown, w.hist_all, sizeof(uint32_t) * per * L, s);
  if (rc == TSA_OK) rc = allgather(comm, sown, w.st_all, sizeof(int32_t) * per, s);
  if (comm->kind == kNccl) {
    const tsa_status rg = nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
    if (rc == TSA_OK) rc = rg;
  }
  SH_TRY(rc);
  // 3. the rank's work units of every slice, merged per slice into its slot
  const int32_t U = tsa_sharded_units(slab, nz_total, P);
  const int32_t u0 = (int32_t)((int64_t)U * r / P), u1 = (int32_t)((int64_t)U * (r + 1) / P);
  double *ms_own = w.ms + (size_t)r * nz_total;
  uint64_t *mk_own = w.mk + (size_t)r * nz_total;
  SH_TRY(cuda(cudaMemcpyAsync(w.st_work, w.st_all, sizeof(int32_t) * nz_total, cudaMemcpyDeviceToDevice, s),
              "status copy"));
  if (u1 > u0) {
    SH_TRY(tsa_search(w.hist_all, w.st_work, nz_total, slab->nx * slab->ny, L, k, slab->q, slab->objective,
                      slab->enumeration, U, u0, u1, w.ps, w.pk, w.search, w.search_bytes, stream));
    SH_TRY(tsa_merge(w.ps, w.pk, u1 - u0, nz_total, ms_own, mk_own, stream));
  } else {
    k_fill_none<<<(unsigned)std::min<int64_t>((nz_total + 255) / 256, 1024), 256, 0, s>>>(ms_own, mk_own, nz_total);
    SH_TRY(cuda(cudaGetLastError(), "k_fill_none"));
  }
  // 4. all-gather the per-rank partials, merge + phi(t*) (identical on every rank)
  if (comm->kind == kNccl) SH_TRY(nccl_check(nccl().GroupStart(), "ncclGroupStart"));
  rc = allgather(comm, ms_own, w.ms, sizeof(double) * nz_total, s);
  if (rc == TSA_OK) rc = allgather(comm, mk_own, w.mk, sizeof(uint64_t) * nz_total, s);
  if (comm->kind == kNccl) {
    const tsa_status rg = nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
    if (rc == TSA_OK) rc = rg;
  }
  SH_TRY(rc);
  tsa_outputs fo = *out;
  fo.labels = nullptr;
  fo.histogram = nullptr;
  if (!fo.slice_status) fo.slice_status = w.st_work;  // (the search is done with it)
  // finalize reads the histogram-pass status (NO_VALID_SPLIT follows from "no key")
  SH_TRY(tsa_finalize(w.hist_all, w.st_all, nz_total, L, k, slab->q, slab->objective, w.ms, w.mk, P, &fo, stream));
  if (out->histogram)
    SH_TRY(cuda(cudaMemcpyAsync(out->histogram, w.hist_all, sizeof(uint32_t) * nz_total * L,
                                cudaMemcpyDeviceToDevice, s), "histogram copy"));
  // 5. labels of the own slab
  if (out->labels && slab->nz > 0) {
    SH_TRY(tsa_label(slab, out->thresholds + z0 * k, fo.slice_status + z0, out->labels, stream));
  }
#undef SH_TRY
  return TSA_OK;
}

}  // extern "C"
