// §8(e) on sm_100a: ONE index built by `world` GPUs with the rows of the N x N
// Eq. 1 matrix sharded across them (north_star "Multi-GPU partitioning: rows
// of the N x N matrix shard naturally across the 8 GPUs of one box").
//
// Rank q owns rows [q*S, min((q+1)*S, M)) of the current matrix (S =
// ceil(M/world)), all columns.  Everything that is O(N) — row keys, the round
// preparation (minimum height, RNN pairs, level cliques, compaction map) — is
// replicated: every rank runs the same kernels on the same data and gets the
// same merges.  The exchanges are fused into the kernels over peer memory
// (CUDA IPC mappings over NVLink/NVSwitch), no collective library:
//   - the distance kernel writes each rank's rows and their NN keys; every
//     rank then copies the other ranks' key slices (k_gather_slices);
//   - a level's adjacency rows are computed by the owner of the row, then
//     copied by every rank from the owners (k_adj_gather);
//   - the compaction kernel (k_merge_rows with PeerRows) builds the new rows
//     a rank owns, reading the member rows from whichever rank holds them,
//     and writes the new keys, which are then gathered like the first ones.
// Ranks meet at a device-side barrier (system-scope atomics on every peer's
// counter) before reading what peers wrote and before a buffer a peer may
// still read is rewritten.  In the single-process mode all `world` ranks live
// on one device with their own buffers and run step by step on one stream
// (barriers are then stream order): the sharded algorithm is validated on one
// GPU against the single-GPU build (tests/test_gpu_parity.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "linkage_kernels.cuh"

namespace ragb {
namespace {

// ---------------------------------------------------------------- layout
size_t take(size_t &o, size_t bytes) {
  const size_t a = (o + 255) & ~(size_t)255;
  o = a + bytes;
  return a;
}

struct DistLayout {
  size_t err, counters, table, idsT, lut, lutc, vals, ptab, key0, key1, rep0, rep1, sz0, sz1, leader, aux0, aux1, aux2, aux3,
      aux4, alive, za, zb, zh, zs, adj, matA, matB, total;
  int64_t S0;  // rows per rank of the distance matrix
  static DistLayout make(int64_t N, int32_t K, int world) {
    DistLayout L{};
    size_t o = 0;
    L.S0 = (N + world - 1) / world;
    L.err = take(o, 64);
    L.counters = take(o, 64);
    L.table = take(o, (size_t)world * 8 * 8);  // device pointer tables (8 x world)
    L.idsT = take(o, (size_t)K * padded_cols(N) * 4);
    {
      int stride;
      int64_t entries;
      distance_lut_layout(K, true, &stride, &entries);
      L.lut = take(o, (size_t)std::max<int64_t>(entries, 1) * 4);
      L.lutc = take(o, (size_t)std::max<int64_t>(entries, 1) * 4);
      L.vals = take(o, (size_t)std::max<int64_t>(entries, 1) * 4);
      L.ptab = take(o, (size_t)tile_ptab_entries(K) * 8);
    }
    L.key0 = take(o, (size_t)(N + world) * 8);
    L.key1 = take(o, (size_t)(N + world) * 8);
    L.rep0 = take(o, (size_t)N * 4);
    L.rep1 = take(o, (size_t)N * 4);
    L.sz0 = take(o, (size_t)N * 4);
    L.sz1 = take(o, (size_t)N * 4);
    L.leader = take(o, (size_t)N * 4);
    L.aux0 = take(o, (size_t)N * 4);
    L.aux1 = take(o, (size_t)(N + 1) * 4);
    L.aux2 = take(o, (size_t)N * 4);
    L.aux3 = take(o, (size_t)(N + 8) * 4);
    L.aux4 = take(o, (size_t)2 * N * 4);
    L.alive = take(o, (size_t)N);
    L.za = take(o, (size_t)N * 4);
    L.zb = take(o, (size_t)N * 4);
    L.zh = take(o, (size_t)N * 4);
    L.zs = take(o, (size_t)N * 4);
    // level adjacency (n x ceil(n/32) words), then the sweep's candidate sets and arrays (linkage_kernels.cuh)
    L.adj = take(o, (2 * (size_t)N * (size_t)((N + 31) / 32) + 6 * (size_t)N) * 4);
    const size_t mat = (size_t)L.S0 * (size_t)((N + 3) & ~3ll) * 4;
    L.matA = take(o, mat);
    L.matB = take(o, mat);
    L.total = (o + 255) & ~(size_t)255;
    return L;
  }
};

template <typename T>
T *at(unsigned char *base, size_t off) {
  return reinterpret_cast<T *>(base + off);
}

// ---------------------------------------------------------------- kernels
// Copy the slices [q*S, min((q+1)*S, M)) of every other rank's array into
// this rank's copy (src[q] = rank q's array, in this process's address space).
template <typename T>
__global__ void k_gather_slices(T *__restrict__ dst, const T *const *__restrict__ src, int world, int self,
                                int64_t S, int64_t M) {
  for (int q = 0; q < world; ++q) {
    if (q == self) continue;
    const T *s = src[q];
    const int64_t a = q * S, b = min((q + 1) * S, M);
    for (int64_t i = a + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x)
      dst[i] = s[i];
  }
}

// Level adjacency rows of the level vertices whose row this rank owns (other
// rows written as zero): adj[i][w] bit j <=> D[list[i]][list[32w + j]] == h.
template <typename T>
__global__ void k_level_adj_dist(PrepArgs a, const T *__restrict__ Dloc, int64_t ld, int64_t r0,
                                 int64_t r1, uint32_t *__restrict__ adj) {
  const int n = a.level[0];
  if (n < 2) return;
  const unsigned hb = (unsigned)a.level[1];
  const int W = (n + 31) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t total = (int64_t)n * W;
  for (int64_t q = gw; q < total; q += nw) {
    const int i = (int)(q / W), w = (int)(q - (int64_t)i * W);
    const int j = w * 32 + lane;
    const int64_t r = a.list[i];
    bool bit = false;
    if (r >= r0 && r < r1 && j < n && j != i) bit = Elem<T>::bits(__ldg(Dloc + (r - r0) * ld + a.list[j])) == hb;
    const unsigned word = __ballot_sync(0xffffffffu, bit);
    if (lane == 0) adj[q] = word;
  }
}

// Copy the adjacency rows owned by other ranks (row i belongs to the owner of
// list[i]; peers hold the same list).
__global__ void k_adj_gather(PrepArgs a, uint32_t *__restrict__ adj, const uint32_t *const *__restrict__ peer_adj,
                             int world, int self, int64_t S) {
  const int n = a.level[0];
  if (n < 2) return;
  const int W = (n + 31) >> 5;
  const int64_t total = (int64_t)n * W;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / W);
    const int owner = (int)(a.list[i] / S);
    if (owner != self) adj[q] = peer_adj[owner][q];
  }
}

// Cross-GPU barrier: signal every rank's counter (system-scope atomics on
// peer memory), wait until this rank's counter reaches `target`.  Bounded
// spin: a peer that never arrives sets err instead of hanging the device.
__global__ void k_barrier(unsigned *const *__restrict__ peer_bar, unsigned *my_bar, int world, unsigned target,
                          unsigned *err) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int q = 0; q < world; ++q) atomicAdd_system(peer_bar[q], 1u);
  const long long t0 = clock64();
  while (atomicAdd_system(my_bar, 0u) < target) {
    if (clock64() - t0 > 40000000000ll) {  // ~20 s
      atomicOr(err, 8u);
      break;
    }
  }
  __threadfence_system();
}

}  // namespace
}  // namespace ragb

// ---------------------------------------------------------------- handle
constexpr int kMaxWorld = 64;

struct rb_dist {
  int world = 1, nlocal = 1, rank0 = 0;
  bool sim = false;                      // all ranks in this process, one device
  std::vector<unsigned char *> scratch;  // [world] rank scratch base (local or IPC-mapped)
  std::vector<float *> rows;             // [world] rank distance-row shard
  std::vector<unsigned *> bar;           // [world] rank barrier counter
  std::vector<size_t> scratch_bytes;     // [world]
  unsigned *my_bar = nullptr;            // cudaMalloc'd by this process (real mode)
  unsigned epoch = 0;
  std::vector<void *> opened;            // IPC mappings to close
  int poison = 0;                        // first CUDA error of a build: the handle is unusable
};

namespace {

rb_status dfail(rb_status code, const std::string &msg);

typedef int (*PFN_getAddressRange)(unsigned long long *, size_t *, unsigned long long);

cudaError_t alloc_base(const void *p, void **base) {
  static PFN_getAddressRange fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *f = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q);
    if (e != cudaSuccess || !f) return e != cudaSuccess ? e : cudaErrorNotSupported;
    fn = reinterpret_cast<PFN_getAddressRange>(f);
  }
  unsigned long long b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, reinterpret_cast<unsigned long long>(p)) != 0) return cudaErrorInvalidValue;
  *base = reinterpret_cast<void *>(b);
  return cudaSuccess;
}

struct HandleBlob {
  cudaIpcMemHandle_t hs, hr, hb;
  uint64_t off_s, off_r, off_b, scratch_bytes;
  int32_t rank, world;
};

}  // namespace

extern "C" rb_status ragb_fail_msg(rb_status code, const char *msg);  // capi.cpp
extern "C" rb_status ragb_cuda_fail(int e, const char *msg);           // capi.cpp (records sticky errors)
extern "C" rb_status ragb_check_poisoned(void);                        // capi.cpp

namespace {
rb_status dfail(rb_status code, const std::string &msg) { return ragb_fail_msg(code, msg.c_str()); }
}  // namespace

extern "C" {

rb_status rb_dist_create(int32_t world, int32_t rank, int32_t local_ranks, rb_dist **out) {
  if (!out || world < 1 || world > kMaxWorld || rank < 0 || rank >= world ||
      !(local_ranks == 1 || (local_ranks == world && rank == 0)))
    return dfail(RB_EINVAL, "world/rank/local_ranks: one rank per process, or all ranks in one process");
  rb_dist *d = new (std::nothrow) rb_dist();
  if (!d) return dfail(RB_ENOMEM, "host allocation failed");
  d->world = world;
  d->nlocal = local_ranks;
  d->rank0 = rank;
  d->sim = local_ranks == world && world > 1;
  d->scratch.assign(world, nullptr);
  d->rows.assign(world, nullptr);
  d->bar.assign(world, nullptr);
  d->scratch_bytes.assign(world, 0);
  if (!d->sim) {
    cudaError_t e = cudaMalloc(&d->my_bar, 256);
    if (e == cudaSuccess) e = cudaMemset(d->my_bar, 0, 256);
    if (e != cudaSuccess) {
      delete d;
      return dfail(RB_ECUDA, std::string("barrier counter: ") + cudaGetErrorString(e));
    }
    d->bar[rank] = d->my_bar;
  }
  *out = d;
  return RB_OK;
}

rb_status rb_dist_workspace_size(int32_t world, int64_t N, int32_t K, size_t *rows_bytes, size_t *scratch_bytes) {
  if (world < 1 || N < 1 || K < 1 || K > 255 || !rows_bytes || !scratch_bytes)
    return dfail(RB_EINVAL, "bad argument");
  const ragb::DistLayout L = ragb::DistLayout::make(N, K, world);
  *rows_bytes = (size_t)L.S0 * (size_t)N * 4;
  *scratch_bytes = L.total;
  return RB_OK;
}

rb_status rb_dist_attach(rb_dist *d, int32_t rank, float *rows_dev, void *scratch_dev, size_t scratch_bytes) {
  if (!d || rank < 0 || rank >= d->world || !rows_dev || !scratch_dev) return dfail(RB_EINVAL, "bad argument");
  if (rank < d->rank0 || rank >= d->rank0 + d->nlocal) return dfail(RB_EINVAL, "rank is not local to this process");
  d->rows[rank] = rows_dev;
  d->scratch[rank] = static_cast<unsigned char *>(scratch_dev);
  d->scratch_bytes[rank] = scratch_bytes;
  return RB_OK;
}

rb_status rb_dist_export(const rb_dist *d, void *blob, size_t blob_bytes) {
  if (!d || !blob || blob_bytes < sizeof(HandleBlob)) return dfail(RB_EINVAL, "bad argument");
  if (d->sim) return dfail(RB_ESTATE, "single-process mode has nothing to export");
  const int r = d->rank0;
  if (!d->scratch[r]) return dfail(RB_ESTATE, "attach the rank's buffers first");
  HandleBlob h{};
  void *bs = nullptr, *br = nullptr, *bb = nullptr;
  cudaError_t e;
  if ((e = alloc_base(d->scratch[r], &bs)) != cudaSuccess || (e = alloc_base(d->rows[r], &br)) != cudaSuccess ||
      (e = alloc_base(d->my_bar, &bb)) != cudaSuccess || (e = cudaIpcGetMemHandle(&h.hs, bs)) != cudaSuccess ||
      (e = cudaIpcGetMemHandle(&h.hr, br)) != cudaSuccess || (e = cudaIpcGetMemHandle(&h.hb, bb)) != cudaSuccess)
    return dfail(RB_ECUDA, std::string("IPC export: ") + cudaGetErrorString(e));
  h.off_s = (uint64_t)(d->scratch[r] - static_cast<unsigned char *>(bs));
  h.off_r = (uint64_t)(reinterpret_cast<unsigned char *>(d->rows[r]) - static_cast<unsigned char *>(br));
  h.off_b = (uint64_t)(reinterpret_cast<unsigned char *>(d->my_bar) - static_cast<unsigned char *>(bb));
  h.scratch_bytes = d->scratch_bytes[r];
  h.rank = r;
  h.world = d->world;
  std::memcpy(blob, &h, sizeof(h));
  return RB_OK;
}

rb_status rb_dist_import(rb_dist *d, const void *blob, size_t blob_bytes) {
  if (!d || !blob || blob_bytes < sizeof(HandleBlob)) return dfail(RB_EINVAL, "bad argument");
  HandleBlob h;
  std::memcpy(&h, blob, sizeof(h));
  if (h.world != d->world || h.rank < 0 || h.rank >= d->world) return dfail(RB_EINVAL, "blob from another world");
  if (h.rank == d->rank0) return RB_OK;  // own buffers
  void *ps = nullptr, *pr = nullptr, *pb = nullptr;
  cudaError_t e;
  if ((e = cudaIpcOpenMemHandle(&ps, h.hs, cudaIpcMemLazyEnablePeerAccess)) != cudaSuccess ||
      (e = cudaIpcOpenMemHandle(&pr, h.hr, cudaIpcMemLazyEnablePeerAccess)) != cudaSuccess ||
      (e = cudaIpcOpenMemHandle(&pb, h.hb, cudaIpcMemLazyEnablePeerAccess)) != cudaSuccess)
    return dfail(RB_ECUDA, std::string("IPC import: ") + cudaGetErrorString(e));
  d->opened.push_back(ps);
  d->opened.push_back(pr);
  d->opened.push_back(pb);
  d->scratch[h.rank] = static_cast<unsigned char *>(ps) + h.off_s;
  d->rows[h.rank] = reinterpret_cast<float *>(static_cast<unsigned char *>(pr) + h.off_r);
  d->bar[h.rank] = reinterpret_cast<unsigned *>(static_cast<unsigned char *>(pb) + h.off_b);
  d->scratch_bytes[h.rank] = h.scratch_bytes;
  return RB_OK;
}

void rb_dist_free(rb_dist *d) {
  if (!d) return;
  for (void *p : d->opened) cudaIpcCloseMemHandle(p);
  if (d->my_bar) cudaFree(d->my_bar);
  delete d;
}

}  // extern "C"

// ---------------------------------------------------------------- the build
namespace ragb {

rb_status build_index_dist(rb_dist *d, const uint32_t *ids_d, const uint8_t *lens_d, int64_t N, int32_t K,
                           const rb_params *p, rb_index **out, std::string *msg) {
  const int world = d->world, nloc = d->nlocal, g0 = d->rank0;
  const DistLayout L = DistLayout::make(N, K, world);
  for (int q = 0; q < world; ++q) {
    if (!d->scratch[q] || !d->rows[q]) {
      *msg = "rank " + std::to_string(q) + " has no buffers (attach / import)";
      return RB_ESTATE;
    }
    if (d->scratch_bytes[q] < L.total) {
      *msg = "scratch of rank " + std::to_string(q) + " too small";
      return RB_EINVAL;
    }
  }
  cudaStream_t st = static_cast<cudaStream_t>(p->stream);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int launches = 0;
  cudaError_t e = cudaSuccess;
#define DC(call, where)                                             \
  do {                                                              \
    if ((e = (call)) != cudaSuccess) {                              \
      *msg = std::string(where) + ": " + cudaGetErrorString(e);     \
      d->poison = (int)e;                                           \
      return RB_ECUDA;                                              \
    }                                                               \
  } while (0)
  const auto t_start = std::chrono::steady_clock::now();
  // device pointer tables in each local rank's scratch, written once: rank q's
  // key0 / key1 / adjacency / matA / matB / distance rows / barrier counter,
  // as addresses in this process (local buffers or IPC mappings)
  enum { TK0 = 0, TK1 = 1, TADJ = 2, TA = 3, TB = 4, TROWS = 5, TBAR = 6 };
  auto table = [&](int r, int which) { return at<void *>(d->scratch[r], L.table) + (size_t)which * world; };
  {
    std::vector<void *> tb((size_t)7 * world);
    for (int q = 0; q < world; ++q) {
      tb[TK0 * world + q] = d->scratch[q] + L.key0;
      tb[TK1 * world + q] = d->scratch[q] + L.key1;
      tb[TADJ * world + q] = d->scratch[q] + L.adj;
      tb[TA * world + q] = d->scratch[q] + L.matA;
      tb[TB * world + q] = d->scratch[q] + L.matB;
      tb[TROWS * world + q] = d->rows[q];
      tb[TBAR * world + q] = d->bar[q];
    }
    for (int l = 0; l < nloc; ++l)
      DC(cudaMemcpy(table(g0 + l, 0), tb.data(), tb.size() * 8, cudaMemcpyHostToDevice), "tables");
  }
  auto barrier = [&]() -> cudaError_t {
    if (d->sim || world == 1) return cudaSuccess;  // one stream: program order is the barrier
    ++d->epoch;
    const int r = g0;
    k_barrier<<<1, 32, 0, st>>>(reinterpret_cast<unsigned *const *>(table(r, TBAR)), d->my_bar, world,
                                d->epoch * (unsigned)world, at<uint32_t>(d->scratch[r], L.err));
    ++launches;
    return cudaGetLastError();
  };

  // ---- a1: validation + transposed staging (replicated) --------------------
  const int64_t Npad = padded_cols(N);
  for (int l = 0; l < nloc; ++l) {
    unsigned char *sc = d->scratch[g0 + l];
    DC(cudaMemsetAsync(sc + L.err, 0, 4, st), "memset");
    DC(launch_validate(ids_d, lens_d, N, K, Npad, at<uint32_t>(sc, L.idsT), at<uint32_t>(sc, L.err), st, &launches),
       "validate");
  }
  uint32_t err_h = 0;
  DC(cudaMemcpyAsync(&err_h, d->scratch[g0] + L.err, 4, cudaMemcpyDeviceToHost, st), "D2H err");
  rb_index *idx = new (std::nothrow) rb_index();
  if (!idx) {
    *msg = "host allocation failed";
    return RB_ENOMEM;
  }
  std::unique_ptr<rb_index> guard(idx);
  HostIndex &H = idx->H;
  H.N = N;
  H.K = K;
  H.alpha_num = p->alpha_num;
  H.alpha_den = p->alpha_den;
  H.ids.resize((size_t)N * K);
  if (lens_d) H.lens.resize((size_t)N);
  DC(cudaMemcpyAsync(H.ids.data(), ids_d, (size_t)N * K * 4, cudaMemcpyDeviceToHost, st), "D2H ids");
  if (lens_d) DC(cudaMemcpyAsync(H.lens.data(), lens_d, (size_t)N, cudaMemcpyDeviceToHost, st), "D2H lens");
  DC(cudaStreamSynchronize(st), "validate sync");
  if (err_h & kErrLen) {
    *msg = "context length not in [1, K]";
    return RB_EINVAL;
  }
  if (err_h & kErrReserved) {
    *msg = "reserved DocId 0xFFFFFFFF";
    return RB_EINVAL;
  }
  if (err_h & kErrDup) {
    *msg = "duplicate DocId within a context";
    return RB_EDUPDOC;
  }
  cudaEvent_t ev[4];
  for (auto &x : ev) cudaEventCreate(&x);
  struct EvGuard {
    cudaEvent_t *e;
    ~EvGuard() {
      for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]);
    }
  } evg{ev};
  cudaEventRecord(ev[0], st);

  // ---- a2-a4: this rank's distance rows + their NN keys --------------------
  // code mode (as in the single-GPU build): each rank also
  // writes the 16-bit value codes of its rows (into its B buffer, the first
  // round's input) and the rounds run on codes
  const Tuning tu = Tuning::from(p);
  // host tree stage threads: every rank of the node runs it (replicated),
  // so one process per GPU shares the cores (15 threads each on 8 ranks would
  // oversubscribe the host ~8x)
  if (tu.host_threads > 0)
    set_host_threads(tu.host_threads);
  else if (nloc < world)  // one process per rank
    set_host_threads(std::max(1, (int)(std::thread::hardware_concurrency() / (unsigned)world) - 1));
  const bool codes = N > 1 && tile_path_ok(K, lens_d == nullptr) && tu.value_codes != 0;
  for (int l = 0; l < nloc; ++l) {
    const int r = g0 + l;
    unsigned char *sc = d->scratch[r];
    DistArgs da{};
    da.ids = ids_d;
    da.lens = lens_d;
    da.idsT = at<uint32_t>(sc, L.idsT);
    da.N = N;
    da.Npad = Npad;
    da.row0 = (int64_t)r * L.S0;
    da.nrows = std::max<int64_t>(0, std::min<int64_t>(L.S0, N - da.row0));
    da.K = K;
    da.an = p->alpha_num;
    da.ad = p->alpha_den;
    da.rows = d->rows[r];
    da.nnkey = at<unsigned long long>(sc, L.key0);
    int stride;
    int64_t entries;
    distance_lut_layout(K, lens_d == nullptr, &stride, &entries);
    if (entries > 0) {
      DC(launch_eq1_lut(at<float>(sc, L.lut), K, stride, entries, p->alpha_num, p->alpha_den, st, &launches),
         "eq1 table");
      da.lut = at<float>(sc, L.lut);
      if (tile_path_ok(K, lens_d == nullptr)) {
        DC(launch_code_table(da.lut, K, stride, entries, at<uint32_t>(sc, L.lutc), at<float>(sc, L.vals),
                             at<int>(sc, L.err + 16), st, &launches),
           "code table");
        da.lutc = at<uint32_t>(sc, L.lutc);
        da.vals = at<float>(sc, L.vals);
        da.ptab = at<const uint2>(sc, L.ptab);
        if (codes) da.codes = at<uint16_t>(sc, L.matB);
      }
    }
    if (da.nrows > 0) DC(launch_distance(da, st, &launches), "distance kernel");
  }
  cudaEventRecord(ev[1], st);
  DC(barrier(), "barrier");
  for (int l = 0; l < nloc; ++l) {
    const int r = g0 + l;
    k_gather_slices<unsigned long long><<<sms, 256, 0, st>>>(
        at<unsigned long long>(d->scratch[r], L.key0),
        reinterpret_cast<const unsigned long long *const *>(table(r, TK0)), world, r, L.S0, N);
    ++launches;
  }
  DC(cudaGetLastError(), "key gather");
  H.nn_idx.resize(N);
  H.nn_d.resize(N);
  std::vector<unsigned long long> keys(N);
  DC(cudaMemcpyAsync(keys.data(), d->scratch[g0] + L.key0, N * 8, cudaMemcpyDeviceToHost, st), "D2H nn");
  DC(cudaStreamSynchronize(st), "nn sync");
  for (int64_t i = 0; i < N; ++i) {
    const unsigned long long k = keys[i];
    H.nn_idx[i] = k == ~0ull ? -1 : (int32_t)(k & 0xffffffffu);
    uint32_t bits = (uint32_t)(k >> 32);
    float f;
    std::memcpy(&f, &bits, 4);
    H.nn_d[i] = k == ~0ull ? __builtin_inff() : f;
  }

  // ---- a5: complete linkage, rows sharded -----------------------------------
  // every rank must have gathered the peers' f32 key slices before any rank
  // rewrites its own slice as code keys below (a slow peer could
  // otherwise read already-converted keys)
  if (codes) DC(barrier(), "barrier");
  H.za.assign(std::max<int64_t>(N - 1, 0), 0);
  H.zb.assign(H.za.size(), 0);
  H.zh.assign(H.za.size(), 0.0f);
  H.zs.assign(H.za.size(), 0);
  std::vector<PrepArgs> pa(nloc);
  for (int l = 0; l < nloc; ++l) {
    unsigned char *sc = d->scratch[g0 + l];
    PrepArgs &a = pa[l];
    a = PrepArgs{};
    a.leader = at<int>(sc, L.leader);
    a.alive = at<uint8_t>(sc, L.alive);
    a.newidx = at<int>(sc, L.aux0);
    a.goff = at<int>(sc, L.aux1);
    a.gmem = at<int>(sc, L.aux2);
    a.colsrc = at<int>(sc, L.aux3);
    a.cnt = at<int>(sc, L.aux4);
    a.cursor = a.cnt + N;
    a.list = a.goff;
    a.candA = a.gmem;
    a.candB = a.colsrc;
    a.za = at<int>(sc, L.za);
    a.zb = at<int>(sc, L.zb);
    a.zs = at<int>(sc, L.zs);
    a.zh = at<float>(sc, L.zh);
    int *counters = at<int>(sc, L.counters);
    a.zcount = counters;
    a.Mn = counters + 1;
    a.level = counters + 2;
    a.cstat = nullptr;
    a.vals = codes ? at<float>(sc, L.vals) : nullptr;
    if (codes) {  // row keys (f32 bits) -> code keys, after the host copy of the NN above
      k_keys_to_codes<<<sms, 256, 0, st>>>(at<unsigned long long>(sc, L.key0), N, a.vals, at<int>(sc, L.err + 16));
      ++launches;
    }
    DC(cudaMemsetAsync(counters, 0, 64, st), "memset");
    k_init_state<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(at<int>(sc, L.rep0), at<int>(sc, L.sz0), N);
    ++launches;
  }
  TreeBuild T;
  std::mutex mu;
  std::condition_variable cv;
  int64_t avail = 0;
  std::vector<int64_t> ends;  // merge count at the end of every round (the replay sorts round by round)
  bool finished = false;
  std::thread worker([&] {
    host_begin(H, T);
    size_t ne = 0;
    std::vector<int64_t> my_ends;
    for (;;) {
      int64_t upto;
      bool fin;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return avail > T.done || finished; });
        upto = avail;
        fin = finished;
        my_ends.assign(ends.begin() + ne, ends.end());
        ne = ends.size();
      }
      for (int64_t e2 : my_ends) host_replay(H, T, e2);
      host_replay(H, T, upto);
      if (!T.ok || (fin && T.done >= upto)) break;
    }
  });
  auto stop_worker = [&] {
    {
      std::lock_guard<std::mutex> lk(mu);
      finished = true;
    }
    cv.notify_one();
    worker.join();
  };
  int M = (int)N, rounds = 0, zdone = 0, par = 0;
  std::vector<cudaEvent_t> merge_ev;
  double merge_bytes = 0.0;
  int merge_launches = 0;
  int64_t S = L.S0, ld = N;
  // current matrix: the fp32 distance shards (rows), then A / B alternately;
  // in code mode the first matrix is the code shard in B (then A / B)
  bool cur_is_rows = !codes, cur_is_A = false;
  rb_status rs = RB_OK;
  while (M > 1) {
    const size_t koff = par ? L.key1 : L.key0, knoff = par ? L.key0 : L.key1;
    for (int l = 0; l < nloc; ++l) {
      const int r = g0 + l;
      unsigned char *sc = d->scratch[r];
      PrepArgs &a = pa[l];
      a.M = M;
      a.key = at<unsigned long long>(sc, koff);
      a.rep = at<int>(sc, par ? L.rep1 : L.rep0);
      a.sz = at<int>(sc, par ? L.sz1 : L.sz0);
      a.rep_n = at<int>(sc, par ? L.rep0 : L.rep1);
      a.sz_n = at<int>(sc, par ? L.sz0 : L.sz1);
      const void *Dloc = cur_is_rows ? static_cast<const void *>(d->rows[r])
                                     : static_cast<const void *>(sc + (cur_is_A ? L.matA : L.matB));
      a.D = Dloc;
      a.ld = ld;
      launch_prep_mark(a, sms, st, &launches);
      const int64_t ra = (int64_t)r * S, rz = std::min<int64_t>((int64_t)(r + 1) * S, M);
      if (codes)
        k_level_adj_dist<uint16_t><<<sms * 4, 256, 0, st>>>(a, static_cast<const uint16_t *>(Dloc), ld, ra, rz,
                                                            at<uint32_t>(sc, L.adj));
      else
        k_level_adj_dist<float><<<sms * 4, 256, 0, st>>>(a, static_cast<const float *>(Dloc), ld, ra, rz,
                                                         at<uint32_t>(sc, L.adj));
      launches += 1;
    }
    if ((e = barrier()) != cudaSuccess) break;
    for (int l = 0; l < nloc; ++l) {
      const int r = g0 + l;
      unsigned char *sc = d->scratch[r];
      k_adj_gather<<<sms * 4, 256, 0, st>>>(pa[l], at<uint32_t>(sc, L.adj),
                                            reinterpret_cast<const uint32_t *const *>(table(r, TADJ)), world, r, S);
      const size_t m1 = std::min<size_t>((size_t)M, (size_t)std::min(1024, kWarpCliqueMaxN));  // staged only on the warp path
      const size_t smem = m1 * ((m1 + 31) / 32) * 4;  // the staged adjacency of levels <= 1024
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_level_cliques, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_level_cliques<<<1, CT, smem, st>>>(pa[l], at<uint32_t>(sc, L.adj));
      launch_prep_compact(pa[l], sms, st, &launches);
      launches += 2;
    }
    if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) break;
    int host_c[2];
    if ((e = cudaMemcpyAsync(host_c, d->scratch[g0] + L.counters, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
      break;
    ++rounds;
    const int z0 = zdone, z1 = host_c[0];
    if (z1 > (int)N - 1 || z1 < z0) {
      e = cudaErrorUnknown;
      break;
    }
    if (z1 > z0) {
      unsigned char *sc = d->scratch[g0];
      const size_t n = (size_t)(z1 - z0);
      cudaMemcpyAsync(H.za.data() + z0, at<int>(sc, L.za) + z0, n * 4, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(H.zb.data() + z0, at<int>(sc, L.zb) + z0, n * 4, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(H.zh.data() + z0, at<float>(sc, L.zh) + z0, n * 4, cudaMemcpyDeviceToHost, st);
      if ((e = cudaMemcpyAsync(H.zs.data() + z0, at<int>(sc, L.zs) + z0, n * 4, cudaMemcpyDeviceToHost, st)) !=
              cudaSuccess ||
          (e = cudaStreamSynchronize(st)) != cudaSuccess)
        break;
      zdone = z1;
      {
        std::lock_guard<std::mutex> lk(mu);
        avail = zdone;
        ends.push_back(zdone);
      }
      cv.notify_one();
    }
    const int Mn = host_c[1];
    if (Mn >= M || Mn < 1) {
      e = cudaErrorUnknown;
      break;
    }
    if (Mn > 1) {
      const int64_t Sn = (Mn + world - 1) / world;
      const int64_t ldn = codes ? mat_ld<uint16_t>(Mn) : mat_ld<float>(Mn);
      const int VW = codes ? Elem<uint16_t>::VW : Elem<float>::VW;
      const bool vec = ld % VW == 0;
      const bool wide = Mn > 20 * 1024;
      const int es = codes ? 2 : 4;  // window slot bytes (Win<T>)
      const int maxW = wide ? 224 * 1024 / es : 20 * 1024;
      const int W = std::min<int>((Mn + VW - 1) / VW * VW, maxW);
      const size_t smem = (size_t)W * es;
      const int nth = wide ? 1024 : 256;
      typedef PeerRows<float> PR;
      typedef PeerRows<uint16_t> PR16;
      auto kf = wide ? (vec ? k_merge_rows<true, 1024, float, PR> : k_merge_rows<false, 1024, float, PR>)
                     : (vec ? k_merge_rows<true, 256, float, PR> : k_merge_rows<false, 256, float, PR>);
      auto kc = wide ? (vec ? k_merge_rows<true, 1024, uint16_t, PR16> : k_merge_rows<false, 1024, uint16_t, PR16>)
                     : (vec ? k_merge_rows<true, 256, uint16_t, PR16> : k_merge_rows<false, 256, uint16_t, PR16>);
      int per_sm = 1;
      if (codes) {
        cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kc, nth, smem);
      } else {
        cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, nth, smem);
      }
      cudaEvent_t me[2];  // compaction timing (rb_stats.merge_ms / merge_bytes, this process's ranks)
      cudaEventCreate(&me[0]);
      cudaEventCreate(&me[1]);
      cudaEventRecord(me[0], st);
      for (int l = 0; l < nloc; ++l) {
        const int r = g0 + l;
        unsigned char *sc = d->scratch[r];
        const int tcur = cur_is_rows ? TROWS : (cur_is_A ? TA : TB);
        const int c0 = (int)std::min<int64_t>((int64_t)r * Sn, Mn), c1 = (int)std::min<int64_t>((int64_t)(r + 1) * Sn, Mn);
        unsigned char *Dn = sc + ((cur_is_rows || !cur_is_A) ? L.matA : L.matB);
        if (c1 > c0) {
          const int grid = std::min<int>(c1 - c0, sms * std::max(per_sm, 1));
          if (codes)
            kc<<<grid, nth, smem, st>>>(PR16{reinterpret_cast<const uint16_t *const *>(table(r, tcur)), (int)S, ld},
                                        M, pa[l].Mn, pa[l].goff, pa[l].gmem, pa[l].colsrc, pa[l].cursor, W, c0, c1,
                                        reinterpret_cast<uint16_t *>(Dn), at<unsigned long long>(sc, knoff));
          else
            kf<<<grid, nth, smem, st>>>(PR{reinterpret_cast<const float *const *>(table(r, tcur)), (int)S, ld}, M,
                                        pa[l].Mn, pa[l].goff, pa[l].gmem, pa[l].colsrc, pa[l].cursor, W, c0, c1,
                                        reinterpret_cast<float *>(Dn), at<unsigned long long>(sc, knoff));
          ++launches;
          // algorithmic bytes of this rank: its new rows' member rows read
          // (M columns each) and the new rows written
          const double es = codes ? 2.0 : 4.0;
          merge_bytes += es * ((double)(c1 - c0) * (double)M * ((double)M / (double)Mn) +
                               (double)(c1 - c0) * (double)Mn);
        }
      }
      cudaEventRecord(me[1], st);
      merge_ev.push_back(me[0]);
      merge_ev.push_back(me[1]);
      ++merge_launches;
      if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) break;
      if ((e = barrier()) != cudaSuccess) break;
      for (int l = 0; l < nloc; ++l) {
        const int r = g0 + l;
        k_gather_slices<unsigned long long><<<sms, 256, 0, st>>>(
            at<unsigned long long>(d->scratch[r], knoff),
            reinterpret_cast<const unsigned long long *const *>(table(r, par ? TK0 : TK1)), world, r, Sn, Mn);
        ++launches;
      }
      if (e != cudaSuccess) break;
      // rank buffers stay valid until every rank has gathered (next barrier)
      cur_is_A = cur_is_rows ? true : !cur_is_A;
      cur_is_rows = false;
      S = Sn;
      ld = ldn;
    }
    par ^= 1;
    M = Mn;
  }
  stop_worker();
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    *msg = std::string("sharded linkage: ") + cudaGetErrorString(e);
    return RB_ECUDA;
  }
  uint32_t err2 = 0;
  cudaMemcpy(&err2, d->scratch[g0] + L.err, 4, cudaMemcpyDeviceToHost);
  if (err2 & 8u) {
    *msg = "cross-GPU barrier timed out (a peer rank did not arrive)";
    return RB_ECUDA;
  }
  if (zdone != N - 1) {
    *msg = "sharded linkage did not finish";
    return RB_ECUDA;
  }
  cudaEventRecord(ev[2], st);
  cudaEventSynchronize(ev[2]);
  float ms = 0;
  cudaEventElapsedTime(&ms, ev[0], ev[1]);
  H.stats.distance_ms = ms;
  cudaEventElapsedTime(&ms, ev[1], ev[2]);
  H.stats.linkage_ms = ms;
  H.stats.linkage_rounds = rounds;
  {
    float mt = 0.f;
    for (size_t i = 0; i + 1 < merge_ev.size(); i += 2) {
      float x = 0.f;
      cudaEventElapsedTime(&x, merge_ev[i], merge_ev[i + 1]);
      mt += x;
    }
    for (auto &x : merge_ev) cudaEventDestroy(x);
    H.stats.merge_ms = mt;
    H.stats.merge_bytes = merge_bytes;
    H.stats.merge_launches = merge_launches;
  }
  H.stats.kernel_launches = launches;
  H.stats.value_codes = codes ? 1 : 0;
  const auto th = std::chrono::steady_clock::now();
  rs = host_finish(H, T, msg);
  if (rs != RB_OK) return rs;
  H.has_linkage = true;
  H.stats.host_ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - th).count();
  H.stats.total_ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  *out = guard.release();
  return RB_OK;
#undef DC
}

}  // namespace ragb

extern "C" rb_status rb_build_index_dist(rb_dist *d, const uint32_t *ids_dev, const uint8_t *lens_dev, int64_t N,
                                         int32_t K, const rb_params *p, rb_index **out) {
  if (!d || !ids_dev || !p || !out) return ragb_fail_msg(RB_EINVAL, "NULL argument");
  if (N < 1 || K < 1 || K > 255) return ragb_fail_msg(RB_EINVAL, "N >= 1, 1 <= K <= 255");
  if (p->alpha_den == 0 || p->alpha_den > 1000 || p->alpha_num > p->alpha_den)
    return ragb_fail_msg(RB_EALPHA, "alpha must be num/den with den <= 1000");
  if (!(p->flags & RB_ALPHA_ANY)) {
    const uint64_t n = p->alpha_num, dd = p->alpha_den;
    if (n * 1000 < dd || n * 100 > dd) return ragb_fail_msg(RB_EALPHA, "alpha outside [0.001, 0.01]");
  }
  if (p->linkage != RB_LINK_COMPLETE) return ragb_fail_msg(RB_EINVAL, "the sharded build runs complete linkage");
  if (ragb_check_poisoned() != RB_OK) return RB_ECUDA;
  if (d->poison)
    return ragb_fail_msg(RB_ECUDA, (std::string("handle poisoned by an earlier CUDA error (") +
                                    cudaGetErrorString((cudaError_t)d->poison) + ")").c_str());
  std::string msg;
  const rb_status s = ragb::build_index_dist(d, ids_dev, lens_dev, N, K, p, out, &msg);
  if (s == RB_ECUDA) {
    if (!d->poison) d->poison = (int)cudaErrorUnknown;  // a timed-out barrier or a lost peer
    return ragb_cuda_fail(d->poison, msg.c_str());
  }
  return s == RB_OK ? s : ragb_fail_msg(s, msg.c_str());
}
