// C-ABI entry points of libragb (include/ragb.h): argument checking, scratch
// carving, stage timing, error mapping, handles and sessions.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <cstring>
#include <new>
#include <string>
#include <unordered_map>
#include <vector>

#include "internal.h"
#include "ragb.h"

using ragb::HostIndex;
using ragb::ScratchLayout;

struct rb_session {
  std::unordered_map<uint32_t, int32_t> seen;  // doc -> turn first prefilled
  std::vector<uint32_t> ctx;                   // turn-0 context ++ novel docs
  int32_t turn = 0;
};

namespace {

thread_local std::string g_err;

rb_status fail(rb_status code, const std::string &msg) {
  g_err = msg;
  return code;
}

// A sticky CUDA error (a faulting kernel) leaves the context unusable: the
// library records it and every later device call fails fast with RB_ECUDA
// naming the first error, instead of reaching the driver again.
std::atomic<int> g_sticky{0};

bool is_sticky(cudaError_t e) {
  switch (e) {
    case cudaErrorIllegalAddress:
    case cudaErrorLaunchFailure:
    case cudaErrorMisalignedAddress:
    case cudaErrorIllegalInstruction:
    case cudaErrorInvalidAddressSpace:
    case cudaErrorInvalidPc:
    case cudaErrorHardwareStackError:
    case cudaErrorAssert:
    case cudaErrorLaunchTimeout:
    case cudaErrorECCUncorrectable:
    case cudaErrorContextIsDestroyed:
      return true;
    default:
      return false;
  }
}

rb_status cuda_fail(cudaError_t e, const char *where) {
  if (is_sticky(e)) {
    int none = 0;
    g_sticky.compare_exchange_strong(none, (int)e);
  }
  return fail(RB_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

rb_status check_poisoned() {
  const int e = g_sticky.load();
  if (e == 0) return RB_OK;
  return fail(RB_ECUDA, std::string("device poisoned by an earlier CUDA error (") +
                            cudaGetErrorString((cudaError_t)e) + "); restart the process");
}

// RB_ASYNC_HOST: wait for the handle's host stage (once) and report its status
rb_status settle(const rb_index *idx) {
  std::lock_guard<std::mutex> lk(idx->host_mu);
  if (idx->host.joinable()) idx->host.join();
  if (idx->host_status != RB_OK) return fail(idx->host_status, idx->host_msg);
  return RB_OK;
}
#define RB_SETTLE(idx)                                 \
  do {                                                 \
    if (rb_status s_ = settle(idx); s_ != RB_OK) return s_; \
  } while (0)

constexpr size_t kAlign = 256;

size_t take(size_t &o, size_t bytes) {
  o = (o + kAlign - 1) / kAlign * kAlign;
  const size_t at = o;
  o += bytes;
  return at;
}

rb_status check_params(int64_t N, int32_t K, const rb_params *p, int64_t *row0, int64_t *nrows) {
  if (!p) return fail(RB_EINVAL, "params is NULL");
  if (N < 1) return fail(RB_EINVAL, "N must be >= 1");
  if (N > (int64_t)0x7ffffffe) return fail(RB_EINVAL, "N too large");
  if (K < 1 || K > 255) return fail(RB_EINVAL, "K must be in [1, 255]");
  if (p->alpha_den == 0 || p->alpha_den > 1000)
    return fail(RB_EALPHA, "alpha_den must be in [1, 1000]");
  if (p->alpha_num > p->alpha_den) return fail(RB_EALPHA, "alpha must be <= 1");
  if (!(p->flags & RB_ALPHA_ANY)) {
    // 1/1000 <= num/den <= 1/100
    const uint64_t n = p->alpha_num, d = p->alpha_den;
    if (n * 1000 < d || n * 100 > d) return fail(RB_EALPHA, "alpha outside [0.001, 0.01]");
  }
  if (p->linkage != RB_LINK_COMPLETE && p->linkage != RB_LINK_INTERSECTION)
    return fail(RB_EINVAL, "unknown linkage");
  *row0 = p->row0;
  *nrows = p->nrows < 0 ? N - p->row0 : p->nrows;
  if (*row0 < 0 || *nrows < 1 || *row0 + *nrows > N) return fail(RB_EINVAL, "bad row range");
  return RB_OK;
}

}  // namespace

namespace ragb {

Tuning Tuning::from(const rb_params *p) {
  Tuning t;
  t.value_codes = p->value_codes;
  t.inplace = p->inplace;
  if (p->inplace_weight > 0.f) t.inplace_weight = p->inplace_weight;
  t.gather = p->gather;
  t.long_lists = p->long_lists;
  t.dist_grid = p->dist_grid;
  t.host_threads = p->host_threads;
  t.trace = p->trace;
  t.side_buffer = p->side_buffer;
  t.nn_cache = p->nn_cache;
  return t;
}

ScratchLayout ScratchLayout::make(int64_t N, int32_t K, bool keep_rows, bool linkage) {
  ScratchLayout L{};
  size_t o = 0;
  L.err = take(o, 64);
  L.counters = take(o, 64);
  L.idsT = take(o, (size_t)K * padded_cols(N) * 4);
  L.nnkey = take(o, (size_t)N * 8);
  L.stage_ids = take(o, (size_t)N * K * 4);
  L.stage_lens = take(o, (size_t)N);
  {
    int stride;
    int64_t entries;
    distance_lut_layout(K, true, &stride, &entries);
    L.lut = take(o, (size_t)std::max<int64_t>(entries, 1) * 4);
    L.lutc = take(o, (size_t)std::max<int64_t>(entries, 1) * 4);
    L.vals = take(o, (size_t)std::max<int64_t>(entries, 1) * 4);
    L.ptab = take(o, (size_t)tile_ptab_entries(K) * 8);
  }
  if (linkage && N > 1) {
    L.key0 = L.nnkey;
    L.key1 = take(o, (size_t)N * 8);
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
    L.pmap = take(o, (size_t)(N + 128) * 8);
    L.za = take(o, (size_t)N * 4);
    L.zb = take(o, (size_t)N * 4);
    L.zh = take(o, (size_t)N * 4);
    L.zs = take(o, (size_t)N * 4);
    L.amask = take(o, (size_t)(N / 32 + 1) * 4);
    L.mlist = take(o, (size_t)N * 4);
    L.tcol = take(o, (size_t)kSideCap * 4);
    L.tslot = take(o, (size_t)N * 4);
    L.dmask = take(o, (size_t)(N / 32 + 1) * 4);
    L.tctl = take(o, 64);
    L.nnkey2 = take(o, (size_t)N * 8);
    L.nnround = take(o, (size_t)N * 4);
    L.colver = take(o, (size_t)N * 4);
    // compacted matrices: at most (N-1) rows with a leading dimension padded to 4
    // (also holds an N x N copy for the intersection linkage with RB_KEEP_ROWS)
    const size_t mat = std::max((size_t)(N - 1) * (size_t)((N + 2) & ~3ll), (size_t)N * N) * 4;
    // code mode: two code matrices of max(N x N, (N-1) x round_up(N, 8)) in the same region
    const size_t cmat = code_mat_bytes(N);
    L.matA = take(o, std::max(mat, 2 * cmat));
    L.codes = L.matA;
    L.mat16 = L.matA + cmat;
    L.matB = keep_rows ? take(o, mat) : 0;
  }
  L.total = (o + kAlign - 1) / kAlign * kAlign;
  return L;
}

}  // namespace ragb

extern "C" {

// error helpers for the other host translation units (hidden: not rb_ entries)
rb_status ragb_fail_msg(rb_status code, const char *msg) { return fail(code, msg); }
rb_status ragb_cuda_fail(int e, const char *msg) { return cuda_fail((cudaError_t)e, msg); }
rb_status ragb_check_poisoned(void) { return check_poisoned(); }

const char *rb_version(void) { return "ragb 0.1.0 (sm_100a)"; }

const char *rb_last_error(void) { return g_err.c_str(); }

rb_status rb_params_init(rb_params *p) {
  if (!p) return fail(RB_EINVAL, "params is NULL");
  std::memset(p, 0, sizeof(*p));
  p->alpha_num = 1;
  p->alpha_den = 200;
  p->linkage = RB_LINK_COMPLETE;
  p->flags = 0;
  p->stream = nullptr;
  p->row0 = 0;
  p->nrows = -1;
  p->value_codes = -1;
  p->inplace = -1;
  p->inplace_weight = 0.f;
  p->gather = -1;
  p->long_lists = -1;
  p->dist_grid = 0;
  p->host_threads = 0;
  p->trace = 0;
  p->side_buffer = -1;
  p->nn_cache = -1;
  return RB_OK;
}

rb_status rb_workspace_size(int64_t N, int32_t K, const rb_params *p, size_t *rows_bytes,
                            size_t *scratch_bytes) {
  if (!rows_bytes || !scratch_bytes) return fail(RB_EINVAL, "NULL output");
  int64_t row0, nrows;
  rb_status s = check_params(N, K, p, &row0, &nrows);
  if (s != RB_OK) return s;
  const bool linkage = !(p->flags & RB_SKIP_LINKAGE) && nrows == N;
  *rows_bytes = (size_t)nrows * (size_t)N * sizeof(float);
  *scratch_bytes = ScratchLayout::make(N, K, (p->flags & RB_KEEP_ROWS) != 0, linkage).total;
  return RB_OK;
}

static rb_status build_common(const uint32_t *ids_dev, const uint8_t *lens_dev, int64_t N, int32_t K,
                              const rb_params *p, float *rows_dev, void *scratch_dev,
                              size_t scratch_bytes, uint8_t *s_dev, uint16_t *D_dev,
                              const uint32_t *ids_host, const uint8_t *lens_host, rb_index **out) {
  using clock = std::chrono::steady_clock;
  const auto t_start = clock::now();
  if (!out) return fail(RB_EINVAL, "out is NULL");
  if (check_poisoned() != RB_OK) return RB_ECUDA;
  int64_t row0, nrows;
  rb_status s = check_params(N, K, p, &row0, &nrows);
  if (s != RB_OK) return s;
  if (!rows_dev || !scratch_dev) return fail(RB_EINVAL, "NULL device buffer");
  if ((p->flags & RB_EMIT_COUNTS) && (!s_dev || !D_dev))
    return fail(RB_EINVAL, "RB_EMIT_COUNTS needs s_dev and D_dev");
  const bool linkage = !(p->flags & RB_SKIP_LINKAGE) && nrows == N;
  const bool keep_rows = (p->flags & RB_KEEP_ROWS) != 0;
  const ScratchLayout L = ScratchLayout::make(N, K, keep_rows, linkage);
  if (scratch_bytes < L.total) return fail(RB_EINVAL, "scratch too small");
  cudaStream_t st = static_cast<cudaStream_t>(p->stream);
  unsigned char *sc = static_cast<unsigned char *>(scratch_dev);

  rb_index *idx = new (std::nothrow) rb_index();
  if (!idx) return fail(RB_ENOMEM, "host allocation failed");
  HostIndex &H = idx->H;
  H.N = N;
  H.K = K;
  H.row0 = row0;
  H.nrows = nrows;
  H.alpha_num = p->alpha_num;
  H.alpha_den = p->alpha_den;
  const ragb::Tuning tu = ragb::Tuning::from(p);
  H.trace = tu.trace != 0;
#ifdef RAGB_HOST_TRACE
  H.trace = true;  // host-stage laps on stderr (variant build for host profiling)
#endif
  ragb::set_host_threads(tu.host_threads);
  int launches = 0;
  cudaError_t e;
  cudaEvent_t ev[4];
  for (auto &x : ev) cudaEventCreate(&x);
  auto cleanup = [&](rb_status code) {
    for (auto &x : ev) cudaEventDestroy(x);
    if (code != RB_OK) delete idx;
    return code;
  };
#define RB_CUDA(call, where)                                              \
  do {                                                                    \
    if ((e = (call)) != cudaSuccess) return cleanup(cuda_fail(e, where)); \
  } while (0)

  // ---- inputs on the device (host entry: copy inside the call) -----------
  const uint32_t *ids_d = ids_dev;
  const uint8_t *lens_d = lens_dev;
  if (ids_host) {  // end-to-end entry: stage the host inputs in scratch
    uint32_t *sid = reinterpret_cast<uint32_t *>(sc + L.stage_ids);
    RB_CUDA(cudaMemcpyAsync(sid, ids_host, (size_t)N * K * 4, cudaMemcpyHostToDevice, st),
            "H2D ids");
    ids_d = sid;
    if (lens_host) {
      uint8_t *sl = sc + L.stage_lens;
      RB_CUDA(cudaMemcpyAsync(sl, lens_host, (size_t)N, cudaMemcpyHostToDevice, st), "H2D lens");
      lens_d = sl;
    }
  }
  if (!ids_d) return cleanup(fail(RB_EINVAL, "ids is NULL"));

  // ---- a1: validate + transposed staging ----------------------------------
  const int64_t Npad = ragb::padded_cols(N);
  uint32_t *err_d = reinterpret_cast<uint32_t *>(sc + L.err);
  uint32_t *idsT = reinterpret_cast<uint32_t *>(sc + L.idsT);
  RB_CUDA(cudaEventRecord(ev[0], st), "event");
  RB_CUDA(cudaMemsetAsync(err_d, 0, 4, st), "memset");
  RB_CUDA(ragb::launch_validate(ids_d, lens_d, N, K, Npad, idsT, err_d, st, &launches), "validate");
  uint32_t err_h = 0;
  RB_CUDA(cudaMemcpyAsync(&err_h, err_d, 4, cudaMemcpyDeviceToHost, st), "D2H err");
  RB_CUDA(cudaStreamSynchronize(st), "validate sync");
  if (err_h & ragb::kErrLen) return cleanup(fail(RB_EINVAL, "context length not in [1, K]"));
  if (err_h & ragb::kErrReserved) return cleanup(fail(RB_EINVAL, "reserved DocId 0xFFFFFFFF"));
  if (err_h & ragb::kErrDup) return cleanup(fail(RB_EDUPDOC, "duplicate DocId within a context"));
  RB_CUDA(cudaEventRecord(ev[1], st), "event");

  // ---- a2-a4: distance rows + fused row NN --------------------------------
  ragb::DistArgs da{};
  da.ids = ids_d;
  da.lens = lens_d;
  da.idsT = idsT;
  da.N = N;
  da.Npad = Npad;
  da.row0 = row0;
  da.nrows = nrows;
  da.K = K;
  da.an = p->alpha_num;
  da.ad = p->alpha_den;
  da.rows = rows_dev;
  da.s_out = (p->flags & RB_EMIT_COUNTS) ? s_dev : nullptr;
  da.D_out = (p->flags & RB_EMIT_COUNTS) ? D_dev : nullptr;
  da.nnkey = reinterpret_cast<unsigned long long *>(sc + L.nnkey);
  da.lut = nullptr;
  da.grid_cap = tu.dist_grid;
  da.long_lists = tu.long_lists != 0;
  // complete linkage on 16-bit value codes whenever the tile
  // path's Eq. 1 table exists; value_codes = 0 keeps the fp32 matrices (testing)
  const bool code_mode = linkage && p->linkage == RB_LINK_COMPLETE && N > 1 &&
                         ragb::tile_path_ok(K, lens_d == nullptr) && tu.value_codes != 0;
  ragb::CodeMode cm{};
  {
    int stride;
    int64_t entries;
    ragb::distance_lut_layout(K, lens_d == nullptr, &stride, &entries);
    if (entries > 0) {
      float *lut = reinterpret_cast<float *>(sc + L.lut);
      RB_CUDA(ragb::launch_eq1_lut(lut, K, stride, entries, p->alpha_num, p->alpha_den, st,
                                   &launches),
              "eq1 table");
      da.lut = lut;
      if (ragb::tile_path_ok(K, lens_d == nullptr)) {
        // the tile kernel's packed table carries the order-preserving codes
        // (its row minimum runs on them); code mode also stores them
        uint32_t *lutc = reinterpret_cast<uint32_t *>(sc + L.lutc);
        float *vals = reinterpret_cast<float *>(sc + L.vals);
        int *ncode = reinterpret_cast<int *>(sc + L.err + 16);
        RB_CUDA(ragb::launch_code_table(lut, K, stride, entries, lutc, vals, ncode, st, &launches), "code table");
        da.lutc = lutc;
        da.vals = vals;
        da.ptab = reinterpret_cast<const uint2 *>(sc + L.ptab);
        if (code_mode) {
          da.codes = reinterpret_cast<uint16_t *>(sc + L.codes);
          cm.codes = da.codes;
          cm.mat16 = reinterpret_cast<uint16_t *>(sc + L.mat16);
          cm.vals = vals;
          cm.ncode = ncode;
        }
      }
    }
  }
  RB_CUDA(ragb::launch_distance(da, st, &launches), "distance kernel");
  RB_CUDA(cudaEventRecord(ev[2], st), "event");
  // host copy of the contexts for the tree stage, while the distance kernel runs
  H.ids.resize((size_t)N * K);
  if (lens_d) H.lens.resize((size_t)N);
  if (ids_host) {
    std::memcpy(H.ids.data(), ids_host, (size_t)N * K * 4);
    if (lens_host) std::memcpy(H.lens.data(), lens_host, (size_t)N);
  } else {
    // the host copy of the contexts (tree stage) comes from the caller's
    // buffer on a side stream while the distance kernel runs (the input is
    // complete: the stream was synchronised after validation)
    cudaStream_t side = nullptr;
    RB_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking), "side stream");
    e = cudaMemcpyAsync(H.ids.data(), ids_d, (size_t)N * K * 4, cudaMemcpyDeviceToHost, side);
    if (e == cudaSuccess && lens_d) e = cudaMemcpyAsync(H.lens.data(), lens_d, (size_t)N, cudaMemcpyDeviceToHost, side);
    if (e == cudaSuccess) e = cudaStreamSynchronize(side);
    cudaStreamDestroy(side);
    if (e != cudaSuccess) return cleanup(cuda_fail(e, "D2H ids"));
  }
  H.nn_idx.resize(nrows);
  H.nn_d.resize(nrows);
  std::vector<unsigned long long> keys(nrows);
  RB_CUDA(cudaMemcpyAsync(keys.data(), da.nnkey + row0, nrows * 8, cudaMemcpyDeviceToHost, st),
          "D2H nn");

  // ---- a5 (device) with the a6 replay pipelined on a host worker ------------
  ragb::LinkageOut lo;
  ragb::TreeBuild T;
  const bool intersection = linkage && p->linkage == RB_LINK_INTERSECTION;
  auto th_join = clock::now();  // start of the host stage (a6-a7)
  if (intersection) {  // NEXT-3: sequential greedy merges in one cooperative kernel
    H.za.assign(N - 1, 0);
    H.zb.assign(N - 1, 0);
    H.zh.assign(N - 1, 0.0f);
    H.zs.assign(N - 1, 0);
    H.sort_merges = false;
    float *mat = rows_dev;
    if (keep_rows && N > 1) {
      mat = reinterpret_cast<float *>(sc + L.matA);
      RB_CUDA(cudaMemcpyAsync(mat, rows_dev, (size_t)N * N * 4, cudaMemcpyDeviceToDevice, st), "copy rows");
    }
    RB_CUDA(ragb::run_linkage_intersection(mat, N, N, K, Npad, idsT, lens_d, da.nnkey, p->alpha_num,
                                           p->alpha_den, scratch_dev, L, st, H.za.data(), H.zb.data(),
                                           H.zh.data(), H.zs.data(), &launches),
            "intersection linkage");
    lo.rounds = (int)(N - 1);
    ragb::host_begin(H, T);
  } else if (linkage) {
    H.za.assign(N - 1, 0);
    H.zb.assign(N - 1, 0);
    H.zh.assign(N - 1, 0.0f);
    H.zs.assign(N - 1, 0);
    std::mutex mu;
    std::condition_variable cv;
    int64_t avail = 0;
    std::vector<int64_t> ends;  // merge count at the end of every round so far (the replay sorts round by round)
    bool finished = false;
    cudaError_t copy_err = cudaSuccess;
    int cur_dev = 0;
    cudaGetDevice(&cur_dev);
    std::vector<std::pair<char, float>> wlog;  // trace 2: worker laps (b begin, c copy, r replay)
    const auto tw0 = clock::now();
    auto wlap = [&](char c) {
      if (tu.trace == 2) wlog.emplace_back(c, std::chrono::duration<float, std::milli>(clock::now() - tw0).count());
    };
    std::thread worker([&] {
      cudaSetDevice(cur_dev);  // a new thread starts on device 0
      wlap('s');
      ragb::host_begin(H, T);  // sorted leaf sets overlap the device work
      wlap('b');
      // the round's merges come from the device on this thread's own
      // non-blocking stream: the launching thread never waits for them
      cudaStream_t cs = nullptr;
      cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
      int64_t have = 0;
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
        if (upto > have) {
          const size_t n = (size_t)(upto - have);
          cudaMemcpyAsync(H.za.data() + have, reinterpret_cast<int32_t *>(sc + L.za) + have, n * 4,
                          cudaMemcpyDeviceToHost, cs);
          cudaMemcpyAsync(H.zb.data() + have, reinterpret_cast<int32_t *>(sc + L.zb) + have, n * 4,
                          cudaMemcpyDeviceToHost, cs);
          cudaMemcpyAsync(H.zh.data() + have, reinterpret_cast<float *>(sc + L.zh) + have, n * 4,
                          cudaMemcpyDeviceToHost, cs);
          cudaMemcpyAsync(H.zs.data() + have, reinterpret_cast<int32_t *>(sc + L.zs) + have, n * 4,
                          cudaMemcpyDeviceToHost, cs);
          const cudaError_t ce = cudaStreamSynchronize(cs);
          if (ce != cudaSuccess) {
            copy_err = ce;
            break;
          }
          have = upto;
          wlap('c');
        }
        for (int64_t e : my_ends) ragb::host_replay(H, T, e);  // round by round
        ragb::host_replay(H, T, upto);
        wlap('r');
        if (!T.ok || (fin && T.done >= upto)) break;
      }
      if (cs) cudaStreamDestroy(cs);
    });
    const cudaError_t le = ragb::run_linkage(
        rows_dev, N, da.nnkey, scratch_dev, L, keep_rows, code_mode ? &cm : nullptr, st, H.za.data(), H.zb.data(),
        H.zh.data(), H.zs.data(), &lo, &launches, [&](int64_t upto) {
          {
            std::lock_guard<std::mutex> lk(mu);
            avail = upto;
            ends.push_back(upto);
          }
          cv.notify_one();
        },
        tu);
    // the device stage ends here; waiting for the replay worker counts as host time
    cudaEventRecord(ev[3], st);  // (an error surfaces at the sync below: the worker must be joined first)
    th_join = clock::now();
    cudaEvent_t lev = nullptr;
    const auto tj = clock::now();
    if (tu.trace == 2) {
      cudaEventCreate(&lev);
      cudaEventRecord(lev, st);
    }
    {
      std::lock_guard<std::mutex> lk(mu);
      finished = true;
    }
    cv.notify_one();
    worker.join();
    if (lev) {
      float a = 0;
      cudaEventSynchronize(lev);
      cudaEventElapsedTime(&a, ev[2], lev);
      std::fprintf(stderr, "[ragb lt] device linkage=%.3f join=%.3f at %.3f |", a,
                   std::chrono::duration<float, std::milli>(clock::now() - tj).count(),
                   std::chrono::duration<float, std::milli>(tj - tw0).count());
      for (auto &w : wlog) std::fprintf(stderr, " %c%.2f", w.first, w.second);
      std::fprintf(stderr, "\n");
      cudaEventDestroy(lev);
    }
    if (le != cudaSuccess) return cleanup(cuda_fail(le, "linkage"));
    if (copy_err != cudaSuccess) return cleanup(cuda_fail(copy_err, "D2H merges"));
  }
  if (!linkage || intersection) RB_CUDA(cudaEventRecord(ev[3], st), "event");
  RB_CUDA(cudaStreamSynchronize(st), "sync");
  if (!linkage || intersection) th_join = clock::now();
  for (int64_t r = 0; r < nrows; ++r) {
    const unsigned long long k = keys[r];
    if (k == ~0ull) {
      H.nn_idx[r] = -1;
      H.nn_d[r] = __builtin_inff();
    } else {
      H.nn_idx[r] = (int32_t)(k & 0xffffffffu);
      uint32_t bits = (uint32_t)(k >> 32);
      float f;
      std::memcpy(&f, &bits, 4);
      H.nn_d[r] = f;
    }
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, ev[0], ev[1]);
  H.stats.validate_ms = ms;
  cudaEventElapsedTime(&ms, ev[1], ev[2]);
  H.stats.distance_ms = ms;
  cudaEventElapsedTime(&ms, ev[2], ev[3]);
  H.stats.linkage_ms = ms;
  H.stats.linkage_rounds = lo.rounds;
  H.stats.merge_ms = lo.merge_ms;
  H.stats.merge_launches = lo.merge_launches;
  H.stats.merge_bytes = lo.merge_bytes;
  H.stats.value_codes = code_mode ? 1 : 0;
  H.stats.max_level = lo.max_level;
  H.stats.paths = (int32_t)lo.paths;
  H.stats.kernel_launches = launches;

  // ---- a6-a7: tree, orders, schedule (host) --------------------------------
  // (RB_ASYNC_HOST: on a library thread after this call returns; the device
  // and the caller's buffers are no longer used by then)
  auto host_stage = [idx, th = th_join, t_start, trace2 = tu.trace == 2](ragb::TreeBuild &TB) -> rb_status {
    HostIndex &HH = idx->H;
    const auto tf = clock::now();
    std::string msg;
    const rb_status hs = ragb::host_finish(HH, TB, &msg);
    if (hs != RB_OK) {
      idx->host_msg = "internal: " + msg;
      return hs;
    }
    HH.has_linkage = true;
    HH.stats.host_ms = std::chrono::duration<float, std::milli>(clock::now() - th).count();
    if (trace2)
      std::fprintf(stderr, "[ragb lt] host stage: to finish %.3f, finish %.3f ms\n",
                   std::chrono::duration<float, std::milli>(tf - th).count(),
                   std::chrono::duration<float, std::milli>(clock::now() - tf).count());
    HH.stats.total_ms = std::chrono::duration<float, std::milli>(clock::now() - t_start).count();
    return RB_OK;
  };
  if (linkage && (p->flags & RB_ASYNC_HOST)) {
    auto tb = std::make_shared<ragb::TreeBuild>(std::move(T));
    try {
      idx->host = std::thread([idx, tb, host_stage]() mutable {
        try {
          idx->host_status = host_stage(*tb);
        } catch (...) {  // (no exception may leave the library's thread)
          idx->host_msg = "host stage: allocation failed";
          idx->host_status = RB_ENOMEM;
        }
      });
    } catch (...) {
      return cleanup(fail(RB_ENOMEM, "host stage thread"));
    }
  } else {
    if (linkage && (s = host_stage(T)) != RB_OK) return cleanup(fail(s, idx->host_msg));
    H.stats.total_ms = std::chrono::duration<float, std::milli>(clock::now() - t_start).count();
  }
  *out = idx;
  g_err.clear();
  return cleanup(RB_OK);
#undef RB_CUDA
}

rb_status rb_build_index(const uint32_t *ids_dev, const uint8_t *lens_dev, int64_t N, int32_t K,
                         const rb_params *p, float *rows_dev, void *scratch_dev, size_t scratch_bytes,
                         uint8_t *s_dev, uint16_t *D_dev, rb_index **out) {
  if (!ids_dev) return fail(RB_EINVAL, "ids_dev is NULL");
  return build_common(ids_dev, lens_dev, N, K, p, rows_dev, scratch_dev, scratch_bytes, s_dev, D_dev,
                      nullptr, nullptr, out);
}

rb_status rb_build_index_host(const uint32_t *ids_host, const uint8_t *lens_host, int64_t N,
                              int32_t K, const rb_params *p, float *rows_dev, void *scratch_dev,
                              size_t scratch_bytes, rb_index **out) {
  if (!ids_host) return fail(RB_EINVAL, "ids_host is NULL");
  return build_common(nullptr, nullptr, N, K, p, rows_dev, scratch_dev, scratch_bytes, nullptr,
                      nullptr, ids_host, lens_host, out);
}

rb_status rb_index_from_linkage(const uint32_t *ids_host, const uint8_t *lens_host, int64_t N,
                                int32_t K, const int32_t *a, const int32_t *b, const float *h,
                                const int32_t *size, rb_index **out) {
  if (!ids_host || !out || (N > 1 && (!a || !b || !h || !size)))
    return fail(RB_EINVAL, "NULL argument");
  if (N < 1 || K < 1 || K > 255) return fail(RB_EINVAL, "bad N/K");
  rb_index *idx = new (std::nothrow) rb_index();
  if (!idx) return fail(RB_ENOMEM, "host allocation failed");
  HostIndex &H = idx->H;
  H.N = N;
  H.K = K;
  H.row0 = 0;
  H.nrows = N;
  H.ids.assign(ids_host, ids_host + (size_t)N * K);
  if (lens_host) H.lens.assign(lens_host, lens_host + N);
  // validate contexts (same rules as the device a1)
  for (int64_t i = 0; i < N; ++i) {
    const int L = lens_host ? lens_host[i] : K;
    if (L < 1 || L > K) {
      delete idx;
      return fail(RB_EINVAL, "context length not in [1, K]");
    }
    std::unordered_map<uint32_t, int> seen;
    for (int k = 0; k < L; ++k) {
      const uint32_t x = H.ids[(size_t)i * K + k];
      if (x == ragb::kReservedDoc) {
        delete idx;
        return fail(RB_EINVAL, "reserved DocId 0xFFFFFFFF");
      }
      if (!seen.emplace(x, k).second) {
        delete idx;
        return fail(RB_EDUPDOC, "duplicate DocId within a context");
      }
    }
  }
  if (N > 1) {
    H.za.assign(a, a + N - 1);
    H.zb.assign(b, b + N - 1);
    H.zh.assign(h, h + N - 1);
    H.zs.assign(size, size + N - 1);
  }
  std::string msg;
#ifdef RAGB_HOST_TRACE
  H.trace = true;  // host-stage laps on stderr (variant build for host profiling)
#endif
  rb_status s = ragb::host_build(H, &msg);
  if (s != RB_OK) {
    delete idx;
    return fail(s, msg);
  }
  H.has_linkage = true;
  *out = idx;
  return RB_OK;
}

rb_status rb_index_size(const rb_index *idx, int64_t *N, int32_t *K) {
  if (!idx) return fail(RB_EINVAL, "NULL index");
  if (N) *N = idx->H.dyn ? ragb::dyn_contexts(idx->H) : idx->H.N;
  if (K) *K = idx->H.K;
  return RB_OK;
}

rb_status rb_index_stats(const rb_index *idx, rb_stats *st) {
  if (!idx || !st) return fail(RB_EINVAL, "NULL argument");
  RB_SETTLE(idx);
  *st = idx->H.stats;
  return RB_OK;
}

rb_status rb_index_shard(const rb_index *idx, int64_t *row0, int64_t *nrows) {
  if (!idx || !row0 || !nrows) return fail(RB_EINVAL, "NULL argument");
  *row0 = idx->H.row0;
  *nrows = idx->H.nrows;
  return RB_OK;
}

rb_status rb_index_counts(const rb_index *idx, int64_t row0, int64_t nrows, uint8_t *s_dev, uint16_t *D_dev) {
  if (!idx || !s_dev || !D_dev) return fail(RB_EINVAL, "NULL argument");
  RB_SETTLE(idx);
  const HostIndex &H = idx->H;
  if (H.dyn) return fail(RB_ESTATE, "index was updated online (the counts cover the built set only)");
  if (row0 < 0 || nrows < 0 || row0 + nrows > H.N) return fail(RB_EINVAL, "bad row range");
  if (nrows == 0) return RB_OK;
  if (rb_status ps = check_poisoned()) return ps;
  // a2 again for the requested rows, in counts mode, from the index's own
  // copy of the contexts: a rows-only build (no linkage) on temporary buffers
  rb_params p;
  rb_params_init(&p);
  p.alpha_num = H.alpha_num;
  p.alpha_den = H.alpha_den;
  p.flags = RB_EMIT_COUNTS | RB_SKIP_LINKAGE | RB_ALPHA_ANY;  // (alpha was checked when the index was built)
  p.row0 = row0;
  p.nrows = nrows;
  size_t rows_bytes = 0, scratch_bytes = 0;
  if (rb_status s = rb_workspace_size(H.N, H.K, &p, &rows_bytes, &scratch_bytes)) return s;
  void *rows = nullptr, *scratch = nullptr;
  cudaError_t e = cudaMalloc(&rows, rows_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&scratch, std::max<size_t>(scratch_bytes, 1));
  if (e != cudaSuccess) {
    cudaFree(rows);
    return cuda_fail(e, "counts buffers");
  }
  rb_index *tmp = nullptr;
  const rb_status s = build_common(nullptr, nullptr, H.N, H.K, &p, static_cast<float *>(rows), scratch,
                                   scratch_bytes, s_dev, D_dev, H.ids.data(),
                                   H.lens.empty() ? nullptr : H.lens.data(), &tmp);
  if (s == RB_OK) {
    // the build ran on the default stream: the caller's buffers are complete
    e = cudaStreamSynchronize(nullptr);
  }
  rb_index_free(tmp);
  cudaFree(rows);
  cudaFree(scratch);
  if (s != RB_OK) return s;
  return e == cudaSuccess ? RB_OK : cuda_fail(e, "counts");
}

rb_status rb_index_nn(const rb_index *idx, int32_t *nn_idx, float *nn_d) {
  if (!idx) return fail(RB_EINVAL, "NULL index");
  RB_SETTLE(idx);
  const HostIndex &H = idx->H;
  if (H.nn_idx.empty()) return fail(RB_ESTATE, "no NN (index built from a linkage)");
  if (nn_idx) std::memcpy(nn_idx, H.nn_idx.data(), H.nn_idx.size() * 4);
  if (nn_d) std::memcpy(nn_d, H.nn_d.data(), H.nn_d.size() * 4);
  return RB_OK;
}

rb_status rb_index_linkage(const rb_index *idx, int32_t *a, int32_t *b, float *h, int32_t *size) {
  if (!idx) return fail(RB_EINVAL, "NULL index");
  RB_SETTLE(idx);
  const HostIndex &H = idx->H;
  if (!H.has_linkage) return fail(RB_ESTATE, "linkage was skipped");
  const size_t n = H.za.size();
  if (a) std::memcpy(a, H.za.data(), n * 4);
  if (b) std::memcpy(b, H.zb.data(), n * 4);
  if (h) std::memcpy(h, H.zh.data(), n * 4);
  if (size) std::memcpy(size, H.zs.data(), n * 4);
  return RB_OK;
}

static int64_t node_count(const HostIndex &H) { return 1 + H.V + H.N; }

rb_status rb_index_tree_info(const rb_index *idx, int64_t *n_nodes, int64_t *prefix_total,
                             int64_t *path_total) {
  if (!idx) return fail(RB_EINVAL, "NULL index");
  RB_SETTLE(idx);
  const HostIndex &H = idx->H;
  if (!H.has_linkage) return fail(RB_ESTATE, "linkage was skipped");
  if (H.dyn) {
    if (n_nodes) *n_nodes = ragb::dyn_nodes(H);
    ragb::dyn_export(H, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, prefix_total,
                     path_total);
    return RB_OK;
  }
  if (n_nodes) *n_nodes = node_count(H);
  if (prefix_total) {
    int64_t t = H.vpre_off[H.V + 1];
    for (int64_t i = 0; i < H.N; ++i) t += H.lens.empty() ? H.K : H.lens[i];
    *prefix_total = t;
  }
  if (path_total) *path_total = (int64_t)H.path.size();
  return RB_OK;
}

rb_status rb_index_tree(const rb_index *idx, int32_t *parent, int32_t *leaf, int32_t *rep,
                        int64_t *prefix_off, uint32_t *prefix_ids, int64_t *path_off,
                        int32_t *path) {
  if (!idx) return fail(RB_EINVAL, "NULL index");
  RB_SETTLE(idx);
  const HostIndex &H = idx->H;
  if (!H.has_linkage) return fail(RB_ESTATE, "linkage was skipped");
  if (H.dyn) {
    ragb::dyn_export(H, parent, leaf, rep, prefix_off, prefix_ids, path_off, path, nullptr, nullptr);
    return RB_OK;
  }
  const int64_t V = H.V, N = H.N, K = H.K;
  if (parent) {
    parent[0] = -1;
    for (int64_t k = 1; k <= V; ++k) parent[k] = H.vparent[k - 1];
    for (int64_t i = 0; i < N; ++i) parent[V + 1 + i] = H.lparent[i];
  }
  if (leaf) {
    for (int64_t k = 0; k <= V; ++k) leaf[k] = -1;
    for (int64_t i = 0; i < N; ++i) leaf[V + 1 + i] = (int32_t)i;
  }
  if (rep) {
    rep[0] = -1;
    for (int64_t k = 1; k <= V; ++k) rep[k] = H.vrep[k - 1];
    for (int64_t i = 0; i < N; ++i) rep[V + 1 + i] = (int32_t)i;
  }
  if (prefix_off || prefix_ids) {
    int64_t o = 0;
    for (int64_t k = 0; k <= V; ++k) {
      const int64_t a = H.vpre_off[k], b = H.vpre_off[k + 1];
      if (prefix_off) prefix_off[k] = o;
      if (prefix_ids) std::memcpy(prefix_ids + o, H.vpre.data() + a, 4 * (size_t)(b - a));
      o += b - a;
    }
    for (int64_t i = 0; i < N; ++i) {
      const int64_t L = H.lens.empty() ? K : H.lens[i];
      if (prefix_off) prefix_off[V + 1 + i] = o;
      if (prefix_ids) std::memcpy(prefix_ids + o, H.ordered.data() + i * K, 4 * (size_t)L);
      o += L;
    }
    if (prefix_off) prefix_off[V + 1 + N] = o;
  }
  if (path_off) std::memcpy(path_off, H.path_off.data(), H.path_off.size() * 8);
  if (path) std::memcpy(path, H.path.data(), H.path.size() * 4);
  return RB_OK;
}

rb_status rb_order_contexts(rb_index *idx, const uint32_t *ids, const uint8_t *lens, int64_t M,
                            int32_t K, uint32_t *out_ids, uint8_t *out_prefix_len,
                            int64_t *out_schedule) {
  if (!idx) return fail(RB_EINVAL, "NULL index");
  RB_SETTLE(idx);
  HostIndex &H = idx->H;
  if (!H.has_linkage) return fail(RB_ESTATE, "linkage was skipped");
  if (K != H.K) return fail(RB_EINVAL, "K must match the index");
  if (ids) {  // online: search + insert + order the new contexts (NEXT-1)
    if (M < 1) return fail(RB_EINVAL, "M must be >= 1");
    std::string msg;
    const rb_status s = ragb::online_order(H, ids, lens, M, K, H.alpha_num, H.alpha_den, out_ids,
                                           out_prefix_len, out_schedule, &msg);
    if (s != RB_OK) return fail(s, msg);
    return RB_OK;
  }
  if (H.dyn) {
    if (M != ragb::dyn_contexts(H)) return fail(RB_EINVAL, "M must match the indexed contexts");
    ragb::dyn_order_all(H, out_ids, out_prefix_len, out_schedule);
    return RB_OK;
  }
  if (M != H.N) return fail(RB_EINVAL, "M must match the indexed contexts");
  if (out_ids) {  // N x K words: copied by the host-stage threads in 1 MB pieces
    const size_t n = H.ordered.size(), piece = 1 << 18;
    const int64_t np = (int64_t)((n + piece - 1) / piece);
#pragma omp parallel for num_threads(ragb::host_threads()) schedule(static)
    for (int64_t q = 0; q < np; ++q) {
      const size_t b = (size_t)q * piece;
      std::memcpy(out_ids + b, H.ordered.data() + b, std::min(piece, n - b) * 4);
    }
  }
  if (out_prefix_len) std::memcpy(out_prefix_len, H.prefix_len.data(), H.prefix_len.size());
  if (out_schedule) std::memcpy(out_schedule, H.schedule.data(), H.schedule.size() * 8);
  return RB_OK;
}

rb_status rb_index_set_online(rb_index *idx, int32_t device) {
  if (!idx) return fail(RB_EINVAL, "NULL index");
  RB_SETTLE(idx);
  if (device < -1 || device > 1) return fail(RB_EINVAL, "device must be -1, 0 or 1");
  if (device == 1 && check_poisoned() != RB_OK) return RB_ECUDA;
  idx->H.online_device = device;
  return RB_OK;
}

rb_status rb_index_set_alpha(rb_index *idx, uint32_t alpha_num, uint32_t alpha_den) {
  if (!idx) return fail(RB_EINVAL, "NULL index");
  RB_SETTLE(idx);
  if (alpha_den == 0 || alpha_den > 1000 || alpha_num > alpha_den)
    return fail(RB_EALPHA, "alpha must be num/den with 1 <= den <= 1000, num <= den");
  idx->H.alpha_num = alpha_num;
  idx->H.alpha_den = alpha_den;
  return RB_OK;
}

static rb_status session_from_docs(const uint32_t *docs, int32_t n, rb_session **out) {
  rb_session *s = new (std::nothrow) rb_session();
  if (!s) return fail(RB_ENOMEM, "host allocation failed");
  s->seen.reserve((size_t)n * 8 + 16);
  for (int32_t k = 0; k < n; ++k) {
    if (!s->seen.emplace(docs[k], 0).second) {
      delete s;
      return fail(RB_EDUPDOC, "duplicate DocId in turn-0 context");
    }
  }
  s->ctx.assign(docs, docs + n);
  *out = s;
  return RB_OK;
}

rb_status rb_session_open(const rb_index *idx, int64_t row, rb_session **out) {
  if (!idx || !out) return fail(RB_EINVAL, "NULL argument");
  RB_SETTLE(idx);
  const HostIndex &H = idx->H;
  if (!H.has_linkage) return fail(RB_ESTATE, "linkage was skipped");
  if (H.dyn) {
    if (row < 0 || row >= ragb::dyn_contexts(H)) return fail(RB_EPATH, "row out of range");
    const auto &o = ragb::dyn_ordered(H, row);
    return session_from_docs(o.data(), (int32_t)o.size(), out);
  }
  if (row < 0 || row >= H.N) return fail(RB_EPATH, "row out of range");
  // follow the stored search path from the root
  int64_t node = 0;
  for (int64_t z = H.path_off[row]; z < H.path_off[row + 1]; ++z) {
    const int32_t step = H.path[z];
    if (node > H.V) return fail(RB_EPATH, "stale search path");
    const int64_t c0 = H.kids_off[node], c1 = H.kids_off[node + 1];
    if (step < 0 || step >= c1 - c0) return fail(RB_EPATH, "stale search path");
    node = H.kids[c0 + step];
  }
  if (node != H.V + 1 + row) return fail(RB_EPATH, "path does not reach the context");
  const int32_t L = H.lens.empty() ? H.K : H.lens[row];
  return session_from_docs(H.ordered.data() + row * H.K, L, out);
}

rb_status rb_session_open_docs(const uint32_t *docs, int32_t n, rb_session **out) {
  if (!out || (n > 0 && !docs) || n < 0) return fail(RB_EINVAL, "bad argument");
  return session_from_docs(docs, n, out);
}

rb_status rb_dedup_turn(rb_session *s, const uint32_t *ids, int32_t n, uint32_t *novel,
                        int32_t *n_novel, uint32_t *ref_doc, int32_t *ref_turn, int32_t *n_ref) {
  if (!s) return fail(RB_ESESSION, "NULL session");
  if (n < 0 || (n > 0 && (!ids || !novel || !ref_doc || !ref_turn)) || !n_novel || !n_ref)
    return fail(RB_EINVAL, "bad argument");
  for (int32_t k = 0; k < n; ++k)  // duplicate check before any state change
    for (int32_t q = 0; q < k; ++q)
      if (ids[q] == ids[k]) return fail(RB_EDUPDOC, "duplicate DocId in retrieval");
  const int32_t turn = s->turn + 1;
  int32_t nn = 0, nr = 0;
  for (int32_t k = 0; k < n; ++k) {
    auto it = s->seen.find(ids[k]);
    if (it == s->seen.end()) {
      novel[nn++] = ids[k];
    } else {
      ref_doc[nr] = ids[k];
      ref_turn[nr] = it->second;
      ++nr;
    }
  }
  for (int32_t k = 0; k < nn; ++k) s->seen.emplace(novel[k], turn);
  s->ctx.insert(s->ctx.end(), novel, novel + nn);
  s->turn = turn;
  *n_novel = nn;
  *n_ref = nr;
  return RB_OK;
}

rb_status rb_session_context(const rb_session *s, uint32_t *out, int32_t cap, int32_t *n) {
  if (!s) return fail(RB_ESESSION, "NULL session");
  if (!n) return fail(RB_EINVAL, "NULL output");
  *n = (int32_t)s->ctx.size();
  if (out) {
    if (cap < *n) return fail(RB_EINVAL, "output capacity too small");
    std::memcpy(out, s->ctx.data(), s->ctx.size() * 4);
  }
  return RB_OK;
}

rb_status rb_dedup_batch(rb_session *const *sessions, int64_t S, const int64_t *turn_session,
                         const uint32_t *ids, const uint8_t *lens, int64_t M, int32_t K, uint32_t *novel,
                         int32_t *n_novel, uint32_t *ref_doc, int32_t *ref_turn, int32_t *n_ref) {
  if (M < 0 || K < 1 || K > 255 || (M > 0 && (!sessions || !turn_session || !ids || !novel || !n_novel ||
                                               !ref_doc || !ref_turn || !n_ref)))
    return fail(RB_EINVAL, "bad argument");
  // validate everything before any state changes
  for (int64_t i = 0; i < M; ++i) {
    const int64_t si = turn_session[i];
    if (si < 0 || si >= S || !sessions[si]) return fail(RB_ESESSION, "row " + std::to_string(i) + ": bad session");
    const int L = lens ? lens[i] : K;
    if (L < 0 || L > K) return fail(RB_EINVAL, "row " + std::to_string(i) + ": length not in [0, K]");
    const uint32_t *r = ids + i * K;
    for (int k = 1; k < L; ++k)
      for (int q = 0; q < k; ++q)
        if (r[q] == r[k]) return fail(RB_EDUPDOC, "row " + std::to_string(i) + ": duplicate DocId");
  }
  // rows grouped by session (stable: a session's turns keep their order);
  // sessions are independent, so the groups run in parallel
  std::vector<int64_t> off(S + 1, 0), order(M);
  for (int64_t i = 0; i < M; ++i) ++off[turn_session[i] + 1];
  for (int64_t q = 0; q < S; ++q) off[q + 1] += off[q];
  {
    std::vector<int64_t> fill(off.begin(), off.end() - 1);
    for (int64_t i = 0; i < M; ++i) order[fill[turn_session[i]]++] = i;
  }
#pragma omp parallel for schedule(dynamic, 64) num_threads(ragb::host_threads())
  for (int64_t q = 0; q < S; ++q) {
    for (int64_t z = off[q]; z < off[q + 1]; ++z) {
      const int64_t i = order[z];
      const int L = lens ? lens[i] : K;
      rb_dedup_turn(sessions[q], ids + i * K, L, novel + i * K, n_novel + i, ref_doc + i * K, ref_turn + i * K,
                    n_ref + i);
    }
  }
  return RB_OK;
}

rb_status rb_session_turn(const rb_session *s, int32_t *turn) {
  if (!s) return fail(RB_ESESSION, "NULL session");
  if (!turn) return fail(RB_EINVAL, "NULL output");
  *turn = s->turn;
  return RB_OK;
}

rb_status rb_index_cache_event(rb_index *idx, int32_t kind, const int32_t *path, int32_t path_len,
                               int64_t n_tokens, int64_t *taken) {
  if (!idx) return fail(RB_EINVAL, "NULL index");
  RB_SETTLE(idx);
  if (!idx->H.has_linkage) return fail(RB_ESTATE, "linkage was skipped");
  if (path_len < 0) return fail(RB_EINVAL, "negative path length");
  std::string msg;
  const rb_status s = ragb::dyn_cache_event(idx->H, kind, path, path_len, n_tokens, taken, &msg);
  return s == RB_OK ? s : fail(s, msg);
}

rb_status rb_index_cache_state(const rb_index *idx, int64_t *seq_len, int64_t *last_access) {
  if (!idx) return fail(RB_EINVAL, "NULL index");
  RB_SETTLE(idx);
  if (!idx->H.dyn) return fail(RB_ESTATE, "no cache events applied yet");
  ragb::dyn_cache_state(idx->H, seq_len, last_access);
  return RB_OK;
}

void rb_session_free(rb_session *s) { delete s; }
void rb_index_free(rb_index *idx) { delete idx; }  // (joins a pending host stage)

rb_status rb_index_wait(rb_index *idx) {
  if (!idx) return fail(RB_EINVAL, "NULL index");
  return settle(idx);
}

}  // extern "C"
