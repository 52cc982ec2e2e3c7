/*
 * ragb.h — C-ABI of the B200-native RAGBoost context index (arXiv 2511.03475).
 *
 * The boundary follows the paper's problem statement: RAGBoost "takes user
 * prompts and their retrieved results, updates the context to enable effective
 * reuse, and then passes the updated context to the inference engine"
 * (Section 3.3).  Citations: PAPER:n = /root/reference/PAPER.md line
 * n; SPEC:n = /root/reference/SPEC.md line n; X# = a reading listed in
 * DESIGN.md "Readings".
 *
 * Conventions (all entry points):
 *   - Every call returns rb_status (0 = RB_OK, < 0 = error) and never throws.
 *     On error, rb_last_error() returns a thread-local message, valid until
 *     the next call on the same thread.
 *   - Input buffers are borrowed for the duration of the call; the library
 *     copies whatever it retains.
 *   - Large device outputs are CALLER-OWNED (allocated by the caller, e.g. with
 *     torch.empty); sizes come from rb_workspace_size().  The index handle
 *     retains rows_dev/scratch_dev pointers only for the duration of
 *     rb_build_index and owns small host results (nn, merge order, tree,
 *     orders) until rb_index_free().
 *   - On any error the outputs are left untouched, except RB_ECUDA which may
 *     leave device buffers partially written.
 *   - "dev" pointers are CUDA device pointers, "host" pointers are host memory.
 *   - DocIds are uint32; 0xFFFFFFFF is reserved (RB_EINVAL if present).
 *
 * Not thread-safe on a single handle; distinct handles may be used from
 * distinct threads.
 */
#ifndef RAGB_H_
#define RAGB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define RB_API __attribute__((visibility("default")))
#else
#define RB_API
#endif

typedef int32_t rb_status;

enum rb_status_code {
  RB_OK = 0,
  RB_EINVAL = -1,    /* null pointer, N < 1, K < 1, K > 255, len not in [1,K],
                        reserved DocId, workspace too small, bad row range     */
  RB_EDUPDOC = -2,   /* duplicate DocId inside one context: p_i(k) would be
                        ambiguous in Eq. 1 (X5)                         */
  RB_EALPHA = -3,    /* alpha outside [1/1000, 1/100] without
                        RB_ALPHA_ANY, or alpha_den == 0 / > 1000                 */
  RB_ENOMEM = -4,    /* host allocation failed                                   */
  RB_ECUDA = -5,     /* CUDA runtime error (no device, launch failure, ...).
                        A sticky error (a faulting kernel) poisons the process:
                        every later device entry returns RB_ECUDA at once,
                        naming the first error.  An RB_ECUDA from
                        rb_build_index_dist also poisons that rb_dist handle.  */
  RB_ENCCL = -6,     /* reserved (the sharded build exchanges over peer memory,
                        DESIGN.md §8; no collective library on the data path)  */
  RB_EPATH = -7,     /* invalid search path / row index          */
  RB_ESESSION = -8,  /* unknown / null session                        */
  RB_ESTATE = -9     /* precondition, e.g. a stage that was skipped             */
};

/* Linkage: the paper says only "iteratively merge the closest pair"
 * (PAPER:335).  X7: complete linkage on the Eq. 1 matrix, tie key
 * (d, min rep, max rep), rep = smallest leaf index (X8); merges exported in
 * ascending key order (X9).
 * RB_LINK_INTERSECTION (NEXT-3, the SPEC:177 reading): a merged cluster is
 * represented by the ascending sorted intersection of its two representatives
 * ("a virtual node whose context is the sorted intersection") and
 * cluster distances are Eq. 1 between representatives; same tie key.  It is
 * not reducible (heights can decrease), so merges are computed sequentially
 * (N-1 greedy steps on the device) and exported in merge order. */
enum rb_linkage { RB_LINK_COMPLETE = 0, RB_LINK_INTERSECTION = 1 };

enum rb_flags {
  RB_EMIT_COUNTS = 1u << 0,   /* also write s_ij (uint8) and the positional sum
                                 D_ij (uint16) rows — parity/debug output     */
  RB_ALPHA_ANY = 1u << 1,     /* accept alpha outside the paper's band         */
  RB_KEEP_ROWS = 1u << 2,     /* linkage must not overwrite rows_dev           */
  RB_SKIP_LINKAGE = 1u << 3,  /* stop after distance rows + row NN (a1-a4)     */
  RB_ASYNC_HOST = 1u << 4     /* rb_build_index / _host: return once the device
                                 stages (a1-a5) are done; the host stage (a6-a7:
                                 tree, orders, schedule) finishes on a library
                                 thread — see rb_index_wait                    */
};

typedef struct rb_params {
  uint32_t alpha_num;   /* alpha = alpha_num / alpha_den exactly (X1); default 1/200 */
  uint32_t alpha_den;   /* 1 <= alpha_den <= 1000                                    */
  int32_t linkage;      /* rb_linkage                                                */
  uint32_t flags;       /* rb_flags                                                  */
  void *stream;         /* cudaStream_t to launch on (NULL = legacy default stream)  */
  int64_t row0;         /* first distance row this call computes (row sharding)     */
  int64_t nrows;        /* number of rows, -1 = all N (linkage needs all rows)      */
  /* Implementation strategy (tuning and testing).  No result depends on these:
   * the GPU tests compare every setting with the oracle bit for bit.
   * rb_params_init sets each one to its automatic default (-1 or 0). */
  int32_t value_codes;    /* -1 auto: the linkage runs on 16-bit value codes for
                             uniform K <= 32 (complete linkage); 0: fp32 matrices  */
  int32_t inplace;        /* -1 cost model; 0 never; 1 every round where allowed   */
  float inplace_weight;   /* cost-model weight of one merge, in row equivalents
                             (0 = default 56)                                      */
  int32_t gather;         /* -1 auto; 0 window compaction only (no row gather)     */
  int32_t long_lists;     /* -1 auto; 0 the general distance kernel for 32<K<=128  */
  int32_t dist_grid;      /* 0 auto; > 0 caps the distance kernel's grid           */
  int32_t host_threads;   /* 0 auto (all cores); > 0 host tree-stage threads       */
  int32_t trace;          /* 1: per-round linkage (synced) + host-stage trace on stderr; 2: per-round events only */
  int32_t side_buffer;    /* -1 auto: in-place rounds on 16-bit codes append merged
                             columns to a transposed side buffer; 0: rewrite the
                             columns in the matrix                                  */
  int32_t nn_cache;       /* -1 auto: in-place rounds keep each rescanned row's
                             second-nearest key; 0: every affected row rescans    */
} rb_params;

/* Per-build statistics (host, filled by rb_build_index). Times are CUDA-event
 * milliseconds on params.stream, except host_ms (host wall clock). */
typedef struct rb_stats {
  float validate_ms;      /* a1: validation + transposed staging                  */
  float distance_ms;      /* a2-a4: distance rows + fused row NN                   */
  float linkage_ms;       /* a5: all linkage rounds (device)                       */
  float host_ms;          /* a6-a7: merge sort + tree + orders + schedule (host)   */
  float total_ms;         /* whole rb_build_index call, host wall clock            */
  int32_t linkage_rounds; /* number of linkage rounds                              */
  int32_t kernel_launches;/* kernels launched by this call                         */
  int64_t n_virtual;      /* virtual (intersection) nodes kept after collapse      */
  int64_t max_depth;      /* maximum leaf path length                              */
  float merge_ms;         /* CUDA-event time of the linkage compaction launches    */
  int32_t merge_launches; /* number of compaction launches                         */
  double merge_bytes;     /* their algorithmic bytes (live rows read, rows written)*/
  int32_t value_codes;    /* 1: the linkage ran on 16-bit value codes written by the
                             distance kernel next to the fp32 rows (uniform K <= 32,
                             complete linkage); 0: on the fp32 rows              */
  int32_t max_level;      /* largest level list of the linkage rounds (vertices at
                             the round's minimum height)                          */
  int32_t paths;          /* kernel variants the linkage ran (RB_PATH_* bits)     */
} rb_stats;

/* rb_stats.paths bits: which implementation variants a build exercised (tests
 * use them to prove that a parity case reaches the path it is meant for). */
enum rb_path_bits {
  RB_PATH_GATHER = 1u << 0,        /* row-gather compaction, 256-thread CTAs      */
  RB_PATH_GATHER_WIDE = 1u << 1,   /* row-gather compaction, 1024-thread CTAs     */
  RB_PATH_WINDOW = 1u << 2,        /* window compaction, 256-thread CTAs          */
  RB_PATH_WINDOW_WIDE = 1u << 3,   /* window compaction, 1024-thread CTAs         */
  RB_PATH_INPLACE = 1u << 4,       /* in-place round                              */
  RB_PATH_CLIQUE_WARP = 1u << 5,   /* level cliques, warp-resident path           */
  RB_PATH_CLIQUE_BLOCK = 1u << 6   /* level cliques, block path (> 4096 vertices) */
};

typedef struct rb_index rb_index;
typedef struct rb_session rb_session;

/* Library version string. */
RB_API const char *rb_version(void);

/* Thread-local message describing the last error on this thread ("" if none). */
RB_API const char *rb_last_error(void);

/* Fill defaults: alpha 1/200 (X1), complete linkage, no flags, default stream,
 * all rows. */
RB_API rb_status rb_params_init(rb_params *p);

/* Caller-owned buffer sizes for rb_build_index(N, K, p):
 *   rows_bytes    — float rows_dev[nrows][N] (nrows from p; 4*nrows*N bytes);
 *   scratch_bytes — device scratch (validation staging, the Eq. 1 table and
 *                   its value-code table, the linkage matrices: either two
 *                   16-bit code matrices of about N^2 entries each (uniform
 *                   K <= 32, complete linkage) or one fp32 ping-pong matrix
 *                   of at most (N-1)^2 floats — two with RB_KEEP_ROWS —, plus
 *                   O(N) state).  The same size covers both forms.
 * Errors: RB_EINVAL on null outputs, N < 1, K not in [1,255]. */
RB_API rb_status rb_workspace_size(int64_t N, int32_t K, const rb_params *p, size_t *rows_bytes,
                                   size_t *scratch_bytes);

/* Build the context index (Section 4.1 "Index creation"):
 *   a1 validate (K in [1,255], 1 <= len <= K, no duplicate / reserved DocId);
 *   a2-a3 all-pairs Eq. 1 distance rows, d_ij = correctly
 *       rounded fp32 of the exact rational (X6), written to rows_dev;
 *   a4 fused row NN nn_i = argmin_{j != i}(d_ij, j);
 *   a5 complete-linkage merge order (X7-X9);
 *   a6 index tree with virtual intersection nodes, collapse (X10-X12),
 *      leaf search paths ("each leaf node records its search path");
 *   a7 offline prefix-first ordering and schedule
 *      (PAPER:446-464).
 * ids_dev  : uint32 [N][K] row-major, device; row i = context i in retrieval
 *            order (most relevant first).  Slots past lens[i] are ignored.
 * lens_dev : uint8 [N] device, or NULL (all contexts have K docs).
 * rows_dev : float [nrows][N] device, caller-owned (rows p->row0 ..).
 *            Overwritten by the linkage unless RB_KEEP_ROWS (the fp32-matrix
 *            linkage uses it as a ping-pong buffer; the code-matrix linkage,
 *            reported by rb_stats.value_codes, leaves it intact).
 * scratch_dev / scratch_bytes : device scratch of rb_workspace_size() bytes.
 * s_dev, D_dev : with RB_EMIT_COUNTS, uint8/uint16 [nrows][N] device outputs
 *            (else ignored, may be NULL).
 * out      : receives a new handle (free with rb_index_free).
 * Partial rows (p->nrows < N) compute rows + NN for that shard only and imply
 * RB_SKIP_LINKAGE.
 * Errors: RB_EINVAL, RB_EDUPDOC, RB_EALPHA, RB_ECUDA, RB_ENOMEM. */
RB_API rb_status rb_build_index(const uint32_t *ids_dev, const uint8_t *lens_dev, int64_t N, int32_t K,
                                const rb_params *p, float *rows_dev, void *scratch_dev,
                                size_t scratch_bytes, uint8_t *s_dev, uint16_t *D_dev,
                                rb_index **out);

/* Same as rb_build_index but ids/lens are HOST buffers: the host->device copy
 * of the inputs happens inside the call (end-to-end path). */
RB_API rb_status rb_build_index_host(const uint32_t *ids_host, const uint8_t *lens_host, int64_t N,
                                     int32_t K, const rb_params *p, float *rows_dev,
                                     void *scratch_dev, size_t scratch_bytes, rb_index **out);

/* Build only the host-side index (a6-a7) from a given merge order (host
 * buffers, N-1 rows of (a < b, h, size) as rb_index_linkage returns).  No
 * device work; used for multi-rank assembly and CPU tests.
 * Errors: RB_EINVAL (inconsistent merges), RB_EDUPDOC. */
RB_API rb_status rb_index_from_linkage(const uint32_t *ids_host, const uint8_t *lens_host, int64_t N,
                                       int32_t K, const int32_t *a, const int32_t *b,
                                       const float *h, const int32_t *size, rb_index **out);

/* N of the index. */
RB_API rb_status rb_index_size(const rb_index *idx, int64_t *N, int32_t *K);

/* Build statistics. */
RB_API rb_status rb_index_stats(const rb_index *idx, rb_stats *st);

/* RB_ASYNC_HOST builds: wait for the handle's host stage (a6-a7, PAPER:335-339
 * tree + §4.1 ordering) and return its status.  The build call returns once
 * the device work is complete and the caller's device buffers (ids, rows,
 * scratch) are free for the next build; the host stage uses only host memory
 * owned by the handle, so a pipelined caller overlaps it with the next build's
 * device stages.  Every other call on the handle (except rb_index_size /
 * rb_index_shard) waits for it first; rb_index_free joins it.  Without the
 * flag this returns RB_OK at once.  Errors: the host stage's (RB_EINVAL for an
 * inconsistent merge list — an internal error). */
RB_API rb_status rb_index_wait(rb_index *idx);

/* The distance rows this index was built for: [row0, row0 + nrows) (all N
 * for a single-GPU build or an index from a merge list). */
RB_API rb_status rb_index_shard(const rb_index *idx, int64_t *row0, int64_t *nrows);

/* Parity output: s_ij (uint8) and the
 * positional sum D_ij (uint16) of Eq. 1 for rows [row0, row0 + nrows) of the
 * indexed contexts, into caller-owned device buffers [nrows][N] — computed
 * again by the distance kernel from the index's copy of the contexts
 * (temporary device buffers, the default stream, synchronised on return).
 * Errors: RB_EINVAL (NULL buffers, bad range), RB_ESTATE (index updated
 * online), RB_ECUDA, RB_ENOMEM. */
RB_API rb_status rb_index_counts(const rb_index *idx, int64_t row0, int64_t nrows, uint8_t *s_dev,
                                 uint16_t *D_dev);

/* Row NN (host, [nrows]): nn_idx = -1 and nn_d = +inf when N == 1. */
RB_API rb_status rb_index_nn(const rb_index *idx, int32_t *nn_idx, float *nn_d);

/* Merge order (host, [N-1]): rep_a < rep_b (smallest leaf indices), height,
 * merged size; ascending by (h, rep_a, rep_b) = the greedy order (X9).
 * RB_ESTATE if the linkage was skipped. */
RB_API rb_status rb_index_linkage(const rb_index *idx, int32_t *a, int32_t *b, float *h,
                                  int32_t *size);

/* Tree sizes: nodes (root = node 0), total prefix ids, total path entries. */
RB_API rb_status rb_index_tree_info(const rb_index *idx, int64_t *n_nodes, int64_t *prefix_total,
                                    int64_t *path_total);

/* Tree export (host).  parent[n_nodes] (-1 for root), leaf[n_nodes] (context
 * index or -1 for the root / virtual nodes), rep[n_nodes] (smallest leaf
 * index below; -1 for root), prefix_off[n_nodes+1] / prefix_ids[prefix_total]
 * = each node's ordered context (X10), path_off[N+1] / path[path_total] =
 * each leaf's search path.  Any output may be NULL.
 * Node numbering: 0 = root; 1..V = the kept virtual nodes in decreasing order
 * of their merge in the linkage's emission order (round by round; within a
 * round the reciprocal-nearest-neighbour pairs by row, then the level cliques
 * in greedy order), so every parent precedes its children; V+1+i = context i.
 * The emission order is deterministic: the same input gives the same numbers
 * on every run (after online insertions, new nodes are appended). */
RB_API rb_status rb_index_tree(const rb_index *idx, int32_t *parent, int32_t *leaf, int32_t *rep,
                               int64_t *prefix_off, uint32_t *prefix_ids, int64_t *path_off,
                               int32_t *path);

/* Context ordering + schedule (Section 5.1
 * Section 5.2).
 * ids == NULL (offline): the indexed contexts; M must equal the number of
 *   indexed contexts (rb_index_size).  out_ids[M][K] (host): matched prefix
 *   then remaining docs in original order; slots past a context's length are
 *   copied from the input unchanged.  out_prefix_len[M]: inherited prefix
 *   length.  out_schedule[M]: execution order over all indexed contexts.
 * ids != NULL (online, NEXT-1): M new contexts (host [M][K], lens host [M] or
 *   NULL) are searched and inserted one after the other (PAPER:371-384:
 *   greedy descent by minimum Eq. 1 distance against each child's ordered
 *   context, stop at a leaf or when all eligible children are equidistant;
 *   readings X15, X20, X21), then ordered; out_schedule is the Section 5.2
 *   schedule of the batch (indices 0..M-1).  The new contexts become indexed
 *   contexts N, N+1, ... (rb_index_tree / rb_session_open see them).
 * Any output may be NULL.  Errors: RB_EINVAL (K or M mismatch, bad length,
 * reserved DocId), RB_EDUPDOC, RB_ESTATE (linkage skipped). */
RB_API rb_status rb_order_contexts(rb_index *idx, const uint32_t *ids, const uint8_t *lens, int64_t M,
                                   int32_t K, uint32_t *out_ids, uint8_t *out_prefix_len,
                                   int64_t *out_schedule);

/* Where the online search (rb_order_contexts with ids != NULL) scores the
 * root's children, the level whose fan-out reaches thousands: device = 1 on
 * the GPU (one kernel per sub-batch of up to 2048 queries computes Eq. 1 of
 * every query against every child of the root as it was when the sub-batch
 * started; children replaced or appended by earlier queries of the sub-batch
 * are scored on the host, so the results equal the sequential host search bit
 * for bit), 0 on the host, -1 (default) the GPU for batches of >= 64 queries
 * against a root of >= 256 children.  The device buffers are owned by the index
 * (freed by rb_index_free).  Errors: RB_EINVAL, RB_ECUDA (poisoned device). */
RB_API rb_status rb_index_set_online(rb_index *idx, int32_t device);

/* Set the Eq. 1 alpha used by online ordering (an index built from a merge
 * list defaults to 1/200, X1).  Errors: RB_EALPHA. */
RB_API rb_status rb_index_set_alpha(rb_index *idx, uint32_t alpha_num, uint32_t alpha_den);

/* Open a multi-turn session whose turn 0 is indexed context `row`: the
 * session follows the leaf's stored search path to the first-turn context
 * and starts its seen set from it (X18).  Errors: RB_EPATH. */
RB_API rb_status rb_session_open(const rb_index *idx, int64_t row, rb_session **out);

/* Open a session from explicit turn-0 docs (host [n]).  Errors: RB_EDUPDOC. */
RB_API rb_status rb_session_open_docs(const uint32_t *docs, int32_t n, rb_session **out);

/* De-duplicate the next turn (Section 6): novel docs in
 * retrieval order; refs = docs already seen with the turn they were first
 * prefilled, in retrieval order; the seen set grows by the novel docs.
 * ids/novel/ref_doc/ref_turn are host [n] (outputs may hold up to n entries).
 * Errors: RB_ESESSION (null session), RB_EDUPDOC, RB_EINVAL. */
RB_API rb_status rb_dedup_turn(rb_session *s, const uint32_t *ids, int32_t n, uint32_t *novel,
                               int32_t *n_novel, uint32_t *ref_doc, int32_t *ref_turn,
                               int32_t *n_ref);

/* The session's cumulative context: the turn-0 context followed by every
 * turn's novel docs in the order they were prefilled ("appended to a copy of
 * the first-turn context state"; X18).  out: host [cap] or NULL
 * (then only *n is set).  Errors: RB_ESESSION, RB_EINVAL (cap < *n). */
RB_API rb_status rb_session_context(const rb_session *s, uint32_t *out, int32_t cap, int32_t *n);

/* NEXT-2: a batch of follow-up turns over many sessions.
 * Row i (host ids [M][K], lens [M] or NULL = K) is the next turn of session
 * sessions[turn_session[i]]; rows of one session are applied in row order,
 * distinct sessions are independent (processed in parallel on the host).
 * Per row the result equals rb_dedup_turn: novel [M][K] (first n_novel[i]
 * valid), ref_doc / ref_turn [M][K] (first n_ref[i] valid).  All rows are
 * validated before any session changes.  Errors: RB_EINVAL, RB_ESESSION
 * (index out of range or NULL handle), RB_EDUPDOC. */
RB_API rb_status rb_dedup_batch(rb_session *const *sessions, int64_t S, const int64_t *turn_session,
                                const uint32_t *ids, const uint8_t *lens, int64_t M, int32_t K,
                                uint32_t *novel, int32_t *n_novel, uint32_t *ref_doc, int32_t *ref_turn,
                                int32_t *n_ref);

/* Current turn number of a session (0 right after open). */
RB_API rb_status rb_session_turn(const rb_session *s, int32_t *turn);

/* ---- NEXT-4: cache events and a prefix-cache simulator --------------------
 * Index update under cache events (Section 4.1 "Index
 * update": a min-heap of active nodes by last access time; evicted tokens are
 * "removed from the least recently used nodes by decrementing their token
 * counts"; SPEC apply_cache_event).  kind RB_CACHE_APPENDED(path, n): n tokens
 * cached at the node reached by path (host [path_len] child indices, as in
 * rb_index_tree paths), access refreshed; RB_CACHE_ACCESSED(path): access
 * refreshed; RB_CACHE_EVICTED(n): tokens taken from the nodes holding tokens
 * in ascending (last access, node id), zero-clamped; a node left with no
 * tokens and no children is detached from its parent (its later siblings'
 * child indices shift by one), and so are ancestors left empty.  *taken (or
 * NULL) receives the tokens actually evicted.  Detached contexts report an
 * empty path; rb_index_tree reports parent -1 for detached nodes.
 * Errors: RB_EPATH (invalid path), RB_EINVAL (n < 0, unknown kind), RB_ESTATE. */
enum rb_cache_event_kind { RB_CACHE_APPENDED = 0, RB_CACHE_ACCESSED = 1, RB_CACHE_EVICTED = 2 };
RB_API rb_status rb_index_cache_event(rb_index *idx, int32_t kind, const int32_t *path, int32_t path_len,
                                      int64_t n_tokens, int64_t *taken);

/* Per-node cache state after cache events: seq_len (host [n_nodes] or NULL;
 * -1 for a detached node) and last access stamps (host [n_nodes] or NULL);
 * n_nodes from rb_index_tree_info.  Errors: RB_ESTATE (no event applied). */
RB_API rb_status rb_index_cache_state(const rb_index *idx, int64_t *seq_len, int64_t *last_access);

/* Document-granularity prefix cache standing in for the inference engine
 * (Section 2.1 "prefix cache ... trie-based implementation";
 * SPEC cache_sim): a trie over DocId edges with a token budget.  A request's
 * hit is its longest cached prefix, the rest is inserted, and
 * least-recently-used leaves outside the request's path are evicted until the
 * budget holds (ties: older node first).  Errors: RB_EINVAL (capacity <= 0,
 * request larger than the capacity, token count <= 0), RB_EDUPDOC. */
typedef struct rb_cache rb_cache;
RB_API rb_status rb_cache_create(int64_t capacity_tokens, rb_cache **out);
/* One request: docs host [n] in prefill order, doc_tokens host [n] or NULL (1
 * token per doc); outputs hit / miss / evicted tokens. */
RB_API rb_status rb_cache_prefill(rb_cache *c, const uint32_t *docs, int32_t n, const int32_t *doc_tokens,
                                  int64_t *hit, int64_t *miss, int64_t *evicted);
/* M requests (host ids [M][K], lens [M] or NULL) served in `order` (host [M],
 * e.g. rb_order_contexts' schedule; NULL = input order), tokens_per_doc each;
 * per-request outputs host [M] indexed by request. */
RB_API rb_status rb_cache_prefill_batch(rb_cache *c, const uint32_t *ids, const uint8_t *lens,
                                        const int64_t *order, int64_t M, int32_t K, int32_t tokens_per_doc,
                                        int64_t *hit, int64_t *miss, int64_t *evicted);
RB_API rb_status rb_cache_resident(const rb_cache *c, int64_t *tokens);
RB_API void rb_cache_free(rb_cache *c);

/* ---- §8(e): one index built by `world` GPUs, rows sharded ----------------
 * Rank q computes rows [q*S, min((q+1)*S, N)) of the Eq. 1 matrix (S =
 * ceil(N/world)) and, every linkage round, the new rows it owns of the
 * compacted matrix, reading member rows from the rank that holds them over
 * peer memory (CUDA IPC, NVLink/NVSwitch); the O(N) round state (keys, level
 * cliques, compaction map) is replicated and the merges are identical on all
 * ranks (north_star "rows of the N x N matrix shard naturally across the 8
 * GPUs of one box").  One process per GPU: local_ranks = 1; every rank
 * attaches its buffers, exports a handle blob, imports every other rank's
 * blob (exchanged by the caller, e.g. torch.distributed), then all ranks call
 * rb_build_index_dist together.  local_ranks = world (rank 0): all ranks in
 * this process on the current device (validation of the sharded algorithm
 * on one GPU).  Buffers per rank: rows [S][N] floats and scratch, sizes from
 * rb_dist_workspace_size.  Complete linkage only.  A rank that never arrives
 * at a barrier makes the others fail with RB_ECUDA after ~20 s (no hang). */
typedef struct rb_dist rb_dist;
#define RB_DIST_HANDLE_BYTES 256
RB_API rb_status rb_dist_create(int32_t world, int32_t rank, int32_t local_ranks, rb_dist **out);
RB_API rb_status rb_dist_workspace_size(int32_t world, int64_t N, int32_t K, size_t *rows_bytes,
                                        size_t *scratch_bytes);
RB_API rb_status rb_dist_attach(rb_dist *d, int32_t rank, float *rows_dev, void *scratch_dev,
                                size_t scratch_bytes);
RB_API rb_status rb_dist_export(const rb_dist *d, void *blob, size_t blob_bytes);
RB_API rb_status rb_dist_import(rb_dist *d, const void *blob, size_t blob_bytes);
/* ids_dev [N][K] / lens_dev [N] on this rank's device (the same contexts on
 * every rank).  Errors as rb_build_index, RB_ESTATE (buffers missing). */
RB_API rb_status rb_build_index_dist(rb_dist *d, const uint32_t *ids_dev, const uint8_t *lens_dev, int64_t N,
                                     int32_t K, const rb_params *p, rb_index **out);
RB_API void rb_dist_free(rb_dist *d);

RB_API void rb_session_free(rb_session *s);
RB_API void rb_index_free(rb_index *idx);

#ifdef __cplusplus
}
#endif
#endif /* RAGB_H_ */
