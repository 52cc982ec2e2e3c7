// Internal interfaces of libragb (not part of the C-ABI; see include/ragb.h).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <utility>
#include <vector>
#include <thread>
#include <mutex>

#include "ragb.h"

namespace ragb {

constexpr uint32_t kReservedDoc = 0xFFFFFFFFu;  // never a DocId; also the empty-slot key

// Error bits raised by the validation kernel (a1).
enum : uint32_t { kErrLen = 1u, kErrDup = 2u, kErrReserved = 4u };

// Column chunk of the distance kernel: 256 threads x 4 columns.
constexpr int kDistThreads = 256;
constexpr int kColsPerThread = 4;
constexpr int kChunk = kDistThreads * kColsPerThread;

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int64_t padded_cols(int64_t N) { return round_up(N, kChunk); }

// ----------------------------------------------------------------- scratch
// Byte layout of the caller-owned scratch buffer (all offsets 256-aligned).
struct ScratchLayout {
  size_t err, idsT, nnkey, stage_ids, stage_lens, lut, lutc, vals, key0, key1, rep0, rep1, sz0, sz1, leader, aux0, aux1, aux2, aux3, aux4,
      alive, za, zb, zh, zs, amask, mlist, counters, matA, matB, total;
  size_t tcol, tslot, dmask, tctl;  // code mode: in-place side buffer maps (linkage.cu)
  size_t nnkey2, nnround, colver;   // in-place second-nearest cache (linkage.cu)
  size_t pmap;         // code mode: int2 [N + 128] new column -> (leader, pair member), or the compact map
  size_t codes, mat16;  // code mode (inside matA): [N][N] codes, then the first compacted code matrix
  size_t ptab;          // tile path: packed Eq. 1 table (value, code << 16) [(K+1) * (K*K/2+1)]
  static ScratchLayout make(int64_t N, int32_t K, bool keep_rows, bool linkage);
};

// Implementation strategy of one build (rb_params' strategy fields, ragb.h).
// No result depends on it; the GPU tests compare every setting with the oracle.
struct Tuning {
  int value_codes = -1;         // -1 auto, 0 fp32 linkage matrices
  int inplace = -1;             // -1 cost model, 0 never, 1 wherever allowed
  float inplace_weight = 56.f;  // cost-model weight of a merge (row equivalents; measured after the 32-bit rescans: C4 flat 48-56, worse from 64; C3 11.0 -> 10.3 ms at 56)
  int gather = -1;              // -1 auto, 0 window compaction only
  int long_lists = -1;          // -1 auto, 0 general kernel for 32 < K <= 128
  int dist_grid = 0;            // 0 auto, > 0 grid cap of the distance kernel
  int host_threads = 0;         // 0 auto
  int trace = 0;                // per-round trace on stderr (1: synced per round, 2: events only)
  int side_buffer = -1;         // -1 auto, 0 in-place column rewrites in the matrix
  int nn_cache = -1;            // -1 auto, 0 no second-nearest cache (every affected row rescans)
  static Tuning from(const rb_params *p);
};

// ----------------------------------------------------------------- kernels
struct DistArgs {
  const uint32_t *ids;   // [N][K] row-major
  const uint8_t *lens;   // [N] or nullptr
  const uint32_t *idsT;  // [K][Npad] transposed, padded with kReservedDoc
  int64_t N, Npad, row0, nrows;
  int32_t K;
  uint32_t an, ad;
  float *rows;                // [nrows][N]
  uint8_t *s_out;             // [nrows][N] or nullptr
  uint16_t *D_out;            // [nrows][N] or nullptr
  unsigned long long *nnkey;  // [N] indexed by global row: (f32 bits << 32) | column
  const float *lut;           // Eq. 1 table d(s, D) for uniform length K, or nullptr
  // code output (tile path only, complete linkage): codes[i][j] = rank of
  // d_ij among the distinct values of the table (lutc[e] = code of lut[e])
  const uint32_t *lutc;       // [lut entries] or nullptr
  const float *vals;          // [ncode] ascending distinct table values
  uint16_t *codes;            // [nrows][N] or nullptr
  const uint2 *ptab = nullptr;  // tile path: packed (value bits, code << 16) table, filled by the launch
  int grid_cap = 0;           // Tuning::dist_grid
  bool long_lists = true;     // Tuning::long_lists != 0
};

// Order-preserving codes of the Eq. 1 table (distance.cu): lutc[e] = number
// of distinct reachable table values below lut[e]; vals[c] = the value of code
// c (strictly ascending); *ncode = their count (device).
cudaError_t launch_code_table(const float *lut, int32_t K, int stride, int64_t entries, uint32_t *lutc,
                              float *vals, int *ncode, cudaStream_t st, int *launches);

// Linkage on 16-bit codes (linkage.cu): codes [N][N] (ld N) from the distance
// kernel, a second buffer for compacted matrices, the code -> value table.
// Bytes of one code matrix region (capi.cpp ScratchLayout; two per build).
inline size_t code_mat_bytes(int64_t N) {
  return (std::max((size_t)N * N, (size_t)(N - 1) * (size_t)((N + 7) & ~7ll)) * 2 + 255) & ~(size_t)255;
}
constexpr int kSideCap = 8192;  // in-place side buffer: slots (dirty columns) between flushes

struct CodeMode {
  uint16_t *codes;
  uint16_t *mat16;
  const float *vals;
  const int *ncode;  // device
};

// Eq. 1 table d(s, D) at index s * stride + D.  Tile path (uniform K <= 32):
// stride = 1 << shift (the packed accumulator is the index); general path
// (uniform K <= kLutMaxK): stride = floor(K^2/2) + 1; variable lengths: none.
constexpr int kLutMaxK = 128;
constexpr int64_t kLutSmemBytes = 20 * 1024;
void distance_lut_layout(int32_t K, bool uniform, int *stride, int64_t *entries);
cudaError_t launch_eq1_lut(float *lut, int32_t K, int stride, int64_t entries, uint32_t an,
                           uint32_t ad, cudaStream_t st, int *launches);
// Fast path (distance_tile.cu): uniform contexts with K <= 32.
bool tile_path_ok(int32_t K, bool uniform);
int tile_lut_shift(int32_t K);
int64_t tile_lut_entries(int32_t K);
int64_t tile_ptab_entries(int32_t K);
cudaError_t launch_distance_tile(const DistArgs &a, cudaStream_t st);
// Long lists (distance_wide.cu): uniform contexts with 32 < K <= 128.
bool wide_path_ok(int32_t K, bool uniform);
cudaError_t launch_distance_wide(const DistArgs &a, cudaStream_t st);

cudaError_t launch_validate(const uint32_t *ids, const uint8_t *lens, int64_t N, int32_t K,
                            int64_t Npad, uint32_t *idsT, uint32_t *err, cudaStream_t st,
                            int *launches);
cudaError_t launch_distance(const DistArgs &a, cudaStream_t st, int *launches);

struct LinkageOut {
  int rounds = 0;
  float merge_ms = 0.f;     // CUDA-event time of the compaction (k_merge_rows) launches
  int merge_launches = 0;
  double merge_bytes = 0;   // their algorithmic bytes: live old rows read + new rows written
  int max_level = 0;        // largest level list
  unsigned paths = 0;       // RB_PATH_* bits
};

// a5: complete linkage on the full rows (rows ld = N) starting from the fused
// row-NN keys.  Merges are produced in a dependency-respecting order, round by
// round, in the device arrays of the scratch layout (za/zb/zh/zs).  Without
// on_round they are copied to the host arrays za/zb/zh/zs ([N-1]) after each
// round; with on_round, on_round(upto) is called after each round with the
// number of final device merges and the caller copies them (used to pipeline
// the host tree build with the device rounds on a worker thread).
// NEXT-3: intersection-representative linkage (ilinkage.cu); rows [N][ld] are
// updated in place, ctxT [K][Npad] holds the contexts (updated in place),
// merges come back to the host arrays in greedy (merge) order.
cudaError_t run_linkage_intersection(float *rows, int64_t ld, int64_t N, int32_t K, int64_t Npad,
                                     uint32_t *ctxT, const uint8_t *lens, unsigned long long *nnkey,
                                     uint32_t an, uint32_t ad, void *scratch, const ScratchLayout &L,
                                     cudaStream_t st, int32_t *za, int32_t *zb, float *zh, int32_t *zs,
                                     int *launches);

cudaError_t run_linkage(float *rows, int64_t N, unsigned long long *nnkey, void *scratch,
                        const ScratchLayout &L, bool keep_rows, const CodeMode *cm, cudaStream_t st,
                        int32_t *za, int32_t *zb, float *zh, int32_t *zs, LinkageOut *out, int *launches,
                        const std::function<void(int64_t)> &on_round, const Tuning &tu);

// ----------------------------------------------------------------- host
struct DynTree;  // online (mutable) form of the tree, online.cpp
struct OnlineDevState;  // device buffers of the online root scores, online_dev.cu
void online_dev_free(OnlineDevState *s);
// NEXT-1 device step: Eq. 1 of M queries (host [M][K], lens or NULL) against
// the root's children (ordered contexts as CSR coff [F+1] / cdocs, leaf flags
// [F]); returns, per query, the eligible children (X15, X20) as (child index,
// d bits) in ent[q * cap ...], their count in cnt[q] (> cap: overflow).
cudaError_t online_root_scores(OnlineDevState **state, const uint32_t *qids, const uint8_t *qlens, int M, int K,
                               const std::vector<int32_t> &coff, const std::vector<uint32_t> &cdocs,
                               const std::vector<uint8_t> &cleaf, uint32_t an, uint32_t ad, int cap,
                               std::vector<int> *cnt, std::vector<uint2> *ent);

// std::allocator without value-initialisation on resize (large host outputs
// that a parallel loop fills completely: no sequential zero-fill first).
template <typename T>
struct NoInitAlloc : std::allocator<T> {
  template <typename U>
  struct rebind {
    using other = NoInitAlloc<U>;
  };
  NoInitAlloc() = default;
  template <typename U>
  NoInitAlloc(const NoInitAlloc<U> &) noexcept {}
  template <typename U>
  void construct(U *) noexcept {}
  template <typename U, typename... A>
  void construct(U *p, A &&...args) {
    ::new ((void *)p) U(std::forward<A>(args)...);
  }
};

struct HostIndex {
  int64_t N = 0;
  int32_t K = 0;
  int64_t row0 = 0, nrows = 0;  // distance rows this index was built for (rb_index_shard)
  std::vector<uint32_t, NoInitAlloc<uint32_t>> ids;  // [N][K] (filled by copies: no zero fill)
  std::vector<uint8_t> lens;  // [N]
  bool has_linkage = false;
  std::vector<int32_t> nn_idx;
  std::vector<float> nn_d;
  std::vector<int32_t> za, zb, zs;
  std::vector<float> zh;
  // tree: node 0 = root, 1..V = kept virtual nodes, V+1+i = leaf (context) i
  int64_t V = 0;
  std::vector<int32_t> vparent, vrep;  // [V] parent node id / rep of virtual node k (k-1)
  std::vector<int64_t> vpre_off;       // [V+2] ordered prefix CSR by node id 0..V
  std::vector<uint32_t> vpre;
  std::vector<int32_t> lparent;        // [N] parent node id of leaf i
  std::vector<int64_t> kids_off;       // [V+2] children CSR over nodes 0..V, rep order
  std::vector<int32_t> kids;
  std::vector<int64_t> path_off;       // [N+1] leaf search paths
  std::vector<int32_t> path;
  // offline orders
  std::vector<uint32_t, NoInitAlloc<uint32_t>> ordered;   // [N][K]
  std::vector<uint8_t> prefix_len;  // [N]
  std::vector<int64_t> schedule;    // [N]
  rb_stats stats{};
  uint32_t alpha_num = 1, alpha_den = 200;
  bool trace = false;       // Tuning::trace (host-stage laps on stderr)
  bool sort_merges = true;  // complete linkage: export ascending key (X9); intersection: merge order
  std::shared_ptr<DynTree> dyn;             // set by the first online update
  int online_device = -1;                   // NEXT-1 root scores: -1 auto, 0 host, 1 device
  OnlineDevState *odev = nullptr;           // their device buffers (freed with the index)
  int64_t online_stats[2] = {0, 0};         // queries scored on the device, (reserved)
  HostIndex() = default;
  HostIndex(const HostIndex &) = delete;
  HostIndex &operator=(const HostIndex &) = delete;
  ~HostIndex() { if (odev) online_dev_free(odev); }
};

// NEXT-1: online search + insert + ordering of M new contexts (online.cpp).
rb_status online_order(HostIndex &H, const uint32_t *ids, const uint8_t *lens, int64_t M, int32_t K,
                       uint32_t an, uint32_t ad, uint32_t *out_ids, uint8_t *out_prefix_len,
                       int64_t *out_schedule, std::string *msg);
int64_t dyn_contexts(const HostIndex &H);
int64_t dyn_nodes(const HostIndex &H);
void dyn_export(const HostIndex &H, int32_t *parent, int32_t *leaf, int32_t *rep, int64_t *prefix_off,
                uint32_t *prefix_ids, int64_t *path_off, int32_t *path, int64_t *prefix_total,
                int64_t *path_total);
rb_status dyn_cache_event(HostIndex &H, int kind, const int32_t *path, int32_t path_len, int64_t n,
                          int64_t *taken, std::string *msg);
void dyn_cache_state(const HostIndex &H, int64_t *seq_len, int64_t *last_access);
const std::vector<uint32_t> &dyn_ordered(const HostIndex &H, int64_t ctx);
void dyn_order_all(const HostIndex &H, uint32_t *out_ids, uint8_t *out_prefix_len,
                   int64_t *out_schedule);

// Sort merges into greedy key order (X9) and validate them; builds tree,
// orders and schedule (a6-a7).  Returns RB_OK or RB_EINVAL with msg.
rb_status host_build(HostIndex &H, std::string *msg);
int host_threads();
void set_host_threads(int n);  // 0 = auto (Tuning::host_threads of the current build)

// Incremental raw-tree replay, so the host tree can be built while the device
// is still running later linkage rounds.
struct MergeKey {  // one merge in the exported (key-sorted, X9) order
  float h;
  int32_t a, b, size;
};
struct TreeBuild {
  std::vector<MergeKey> zk;     // merges replayed so far, each round's batch sorted by key
  std::vector<int64_t> runs;    // boundaries of the sorted batches in zk
  std::vector<int64_t> rpar;    // [N + N-1] raw parent node of every node (-1: none yet)
  std::vector<uint8_t> keep;    // [N-1] raw merge t kept by the collapse (X11), set once its parent exists
  std::vector<uint32_t, NoInitAlloc<uint32_t>> lset;  // [N][K] sorted leaf sets (written by the sort threads: no fill)
  std::vector<int64_t> voff;    // [N] offsets of merge t's intersection set
  std::vector<uint32_t> vpool;
  std::vector<int32_t> rchild;  // [2(N-1)] raw children of merge t
  std::vector<int32_t> cur, csize;
  int64_t done = 0;
  bool ok = true;
  std::string err;
};
void host_begin(HostIndex &H, TreeBuild &T);
void host_replay(HostIndex &H, TreeBuild &T, int64_t upto);
rb_status host_finish(HostIndex &H, TreeBuild &T, std::string *msg);

}  // namespace ragb

// the C-ABI handle (capi.cpp, dist.cu)
struct rb_index {
  ragb::HostIndex H;
  // RB_ASYNC_HOST: the host stage (a6-a7) runs on `host` after the build call
  // returned; every call on the handle settles it first (capi.cpp settle())
  mutable std::mutex host_mu;
  mutable std::thread host;
  mutable rb_status host_status = RB_OK;
  mutable std::string host_msg;
  ~rb_index() {
    if (host.joinable()) host.join();
  }
};
