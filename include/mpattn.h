/*
 * libmpattn -- B200 (sm_100a) kernels for the Multipole Attention decode path.
 *
 * C ABI: plain device pointers, sizes and a cudaStream_t passed as void*.  Every entry
 * point is stream-ordered, graph-capturable, allocates nothing, and returns 0 on
 * success or a nonzero code (see MPA_ERR_*; CUDA errors are returned as their
 * cudaError_t value) with a message available from mpa_last_error().
 *
 * Data layout ("ledger" l = seq * n_kv_heads + kv_head, L ledgers, head_dim d):
 *   KV cache      k_rot / k_raw / v : [L, tcap, d]  (dtype MPA_F32 or MPA_BF16)
 *   fine level    kc / vc           : [L, kcap, d]  (serving dtype), size [L, kcap],
 *                 count [L], mem_off [L, kcap + 1] (CSR into mem), mem [L, tcap]
 *   coarse level  kc / vc           : [L, ccap, d], size [L, ccap], count [L],
 *                 child_off [L, ccap + 1] (CSR into child), child [L, kcap]
 *
 * Each entry point names the reference function it replaces
 * (/root/reference/pkg/src/multipole_attn/<file>:<line>).
 */
#ifndef MPATTN_H
#define MPATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { MPA_F32 = 0, MPA_BF16 = 1, MPA_F64 = 2 /* centroid levels only */ };

enum {
    MPA_OK = 0,
    MPA_ERR_ARG = 1001,       /* bad argument (shape, dtype, null pointer) */
    MPA_ERR_UNSUPPORTED = 1002 /* configuration the kernels do not implement */
};

/* Last error message of the calling thread ("" if none). */
const char* mpa_last_error(void);
/* Library version string and the sm architecture it was compiled for. */
const char* mpa_version(void);

typedef struct mpa_cache {
    void* k_rot;      /* keys rotated at their true positions (exact-attention view) */
    void* k_raw;      /* pre-rotation keys (clustering / windowed lookup view), [L, tcap, d] */
    void* v;
    int32_t dtype;
    int32_t n_ledgers;
    int32_t tcap;
    int32_t head_dim;
    /* Paged serving cache (block_table != NULL; pipeline.py:26-52 `_KvStore` as a page pool):
     * k_rot and v are pools [n_pages, n_kv_heads, page_size, d] (the HND block layout of paged
     * decode kernels: a head's tokens are contiguous inside a page) and token t of ledger
     * l = s * n_kv_heads + h lives in row (block_table[s, t / page_size] * n_kv_heads + h) *
     * page_size + t % page_size.  k_raw (the clustering view) stays [L, tcap, d].
     * block_table == NULL: k_rot / v are [L, tcap, d] like k_raw. */
    const int32_t* block_table;  /* [n_seq, pages_per_seq] physical page ids */
    int32_t page_size;           /* tokens per page, a power of two */
    int32_t pages_per_seq;
    int32_t n_pages;
    int32_t n_kv_heads;
} mpa_cache;

typedef struct mpa_level {
    const void* kc;          /* [L, cap, d] key centroids: serving dtype, or fp64 (MPA_F64) */
    const void* vc;          /* [L, cap, d] value centroids               */
    const int32_t* size;     /* [L, cap]                                   */
    const int32_t* count;    /* [L]                                        */
    const int32_t* off;      /* [L, cap + 1] CSR offsets (members or children) */
    const int32_t* idx;      /* [L, idx_cap] member token ids or child fine ids */
    int32_t cap;
    int32_t idx_cap;
    int32_t dtype;           /* dtype of kc; vc always has the KV-cache dtype */
    int32_t n_ledgers;
} mpa_level;

/* K1/K14 -- write n_tok new tokens per ledger at positions pos0[l] .. pos0[l]+n_tok-1:
 * k_raw = k, v = v, k_rot = rotate(k, pos) with fp64 angles pos * inv_freq[i]
 * (replaces rope.py:37-53 applied at attention.py:84-85, and pipeline.py:38-44, 156-159).
 * k_src / v_src: fp32 [L, n_tok, d] (device). inv_freq: fp64 [d/2] (device). */
int mpa_kv_write(const mpa_cache* cache, const float* k_src, const float* v_src,
                 const int32_t* pos0, int n_tok, const double* inv_freq, void* stream);

/* K14 -- append n_tok tokens per ledger at the end of each sequence: positions
 * cache_len[l / n_kv_heads] + t (same writes as mpa_kv_write); then cache_len[s] += n_tok and, if
 * given, ntok_dense[l] += n_tok, done on the device by the last block (ticket: one int32
 * workspace, zero-initialised once, left zeroed) -- pipeline.py:156-159 without a host round trip. */
int mpa_kv_append(const mpa_cache* cache, const float* k_src, const float* v_src, int n_kv_heads, int n_tok,
                  int32_t* cache_len, int32_t* ntok_dense, const double* inv_freq, int32_t* ticket,
                  void* stream);

/* Step-input staging: copies three fp32 device buffers (a decode step's q, k, v into the buffers
 * a captured step graph reads) in one launch.  Sizes in elements; any may be 0. */
int mpa_stage3(float* dst0, const float* src0, long long n0, float* dst1, const float* src1, long long n1,
               float* dst2, const float* src2, long long n2, void* stream);

/* Rebind a captured step graph (cudaGraph_t + its cudaGraphExec_t, containing one mpa_decode_step
 * launch) to new q / k_new / v_new device buffers (fp32, 16-byte aligned, the captured shapes): the
 * next launch of the exec reads them directly -- no staging copy per step. */
int mpa_decode_step_rebind(void* graph, void* graph_exec, const float* q, const float* k_new, const float* v_new);

/* One batched serving step from HOST buffers (pinned for overlap), all on `stream`: q, k, v copied
 * into the captured step graph's input block d_in (q, then k, then v, back to back), the graph
 * (cudaGraphExec_t) launched, the output copied back to h_out.  Replaces the per-step host work of
 * the reference's pipeline.step (pipeline.py:124-159) for a whole batch; sizes in bytes. */
int mpa_step_host(void* graph_exec, void* d_in, const void* h_q, long long q_bytes, const void* h_k,
                  long long k_bytes, const void* h_v, long long v_bytes, void* h_out, const void* d_out,
                  long long out_bytes, void* stream);

/* K1 -- rotate queries: q_rot = rotate(q, qpos[seq]) * scale (fp32, exact view) and
 * q_lk = rotate(q, delta) (fp64, lookup view; rope.py:66-68).  q: fp32 [n_seq, n_qh, d].
 * Either output may be NULL (not both): the views are independent. */
int mpa_rotate_queries(const float* q, int n_seq, int n_qh, int d, const int32_t* qpos,
                       int delta, const double* inv_freq, float scale,
                       float* q_rot, double* q_lk, void* stream);

/* K9 -- centroid lookup logits, fp64: logits[l, g, i] = q_lk[seq, h*G+g] . kc[l, id_i] / sqrt(d)
 * for candidates i < n_cand[l]; id_i = cand[l, i] (cand may be NULL: id_i = i, n = lv->count)
 * (attention.py:267-276 `_scores_per_group` logits).  chunk_stats (optional, d in {64,128}):
 * [L, ceil(cap/128), G, 2] per-128-candidate (m_c = max_g l, Z_c = sum N e^(l - m_c)) partials of
 * the normaliser.  e_local (optional, bf16 centroids only): [L, G, cand_cap] e^(l - m_c), which
 * lets the selection form e^(l - max) = e_local e^(m_c - max) without per-candidate exps.
 * n_max (0: cap) bounds the live candidates of every ledger (sizes the grid).
 * rej_w (optional; flat level, bf16, d = 128, with chunk_stats): [L, rej_cap, GP] fp32 replacement
 * weights of EVERY candidate, rej_w[l, i, g] = logit + ln(size) -- the contiguous-centroid work
 * list of mpa_select_worklist (rej == NULL) then masks the selected ones; with rej_w the fp64
 * logits output is optional (NULL: not written -- the selection reads e_local and chunk_stats).
 * q_lk == NULL (bf16, d = 128): the kernel forms the lookup view itself from the fp32 queries q_raw
 * [n_seq, Hq, d] and cs_lk [d/2][2] = (cos, sin)(delta * inv_freq) -- the rotation kernel leaves the
 * critical path. */
int mpa_centroid_logits(const double* q_lk, int n_kv_heads, int group, int d,
                        const mpa_level* lv, const int32_t* cand, const int32_t* n_cand,
                        int cand_cap, double* logits, double* chunk_stats, double* e_local, int n_max,
                        float* rej_w, int rej_cap, const float* q_raw, const double* cs_lk, void* stream);

/* K10 -- Eq. 1 scores and budgeted greedy selection (attention.py:192-207, 267-290).
 * Scores: e_g,i = exp(l_g,i - max_g), Z_g = sum over candidates AND live extras of N * e,
 * score_i = mean_g e_g,i / Z_g.  Selection: visit candidates by (score desc, tie key asc),
 * take while the running size sum < budget[l] (the crossing cluster is included).
 * sizes: lv_size[l, id_i]; tie key: id_i.  Extras (may be NULL): logits [L, G, ecap] with sizes
 * esize[l, j] that enter only the denominators when eflag[l, j] == 0 (hierarchical union,
 * attention.py:331-334).  Writes flag[l, i] = 1 selected / 0 rejected, sel_tokens[l].
 * n_max (<= cand_cap, 0 = cand_cap) bounds the live candidates per ledger (at most 11264) and
 * sizes the shared memory; the crossing candidate is found by a size-weighted radix select on
 * the 64-bit score key then the id.  chunk_stats / e_local: the outputs of mpa_centroid_logits
 * (both optional). */
int mpa_select(const double* logits, int group, const int32_t* cand, const int32_t* n_cand,
               int cand_cap, const int32_t* lv_size, int lv_cap,
               const double* elogits, const int32_t* esize, const uint8_t* eflag,
               const int32_t* n_extra, int ecap,
               const int64_t* budget, int n_ledgers, uint8_t* flag, int32_t* sel_tokens,
               const double* chunk_stats, const double* e_local, int n_max, void* stream);

/* Hierarchy stage glue (attention.py:321-329): cand[l] = children of coarse clusters with
 * cflag == 1, promoted in coarse-id order, children ascending; n_cand[l]. */
int mpa_hier_candidates(const mpa_level* coarse, const uint8_t* cflag, int n_ledgers,
                        int32_t* cand, int32_t* n_cand, int cand_cap, void* stream);


/* K1 + K9 + K10 + work lists + the K/V append of a flat serving decode step in ONE launch (bf16
 * cache and centroids, head_dim 128, 3 <= G <= 8): replaces rope.py:37-53 / 66-68 (exact and
 * lookup views), attention.py:267-290 (`_scores_per_group`), :192-207 (`select_clusters`),
 * :354-375 (`flat_lookup`), the per-kv-head lists of :469-496, and pipeline.py:156-159.
 * One thread-block cluster per ledger (size picked so the grid is one wave): fp64 logits of the
 * lookup view formed from the fp32 queries q [n_seq, Hq, 128] and cs_lk [64][2] = (cos, sin)(delta *
 * inv_freq); per-head max and Z = sum N e^(l - max) over distributed shared memory; Eq. 1 scores;
 * a size-weighted radix select of the crossing candidate (ties: lowest cluster id).  Writes
 * flag [L, cap], sel_tokens [L], tok [L, tok_cap] (sinks ++ buffer ++ members of the selected
 * clusters), stats [4, L] (tokens, rejected centroids, selected tokens, selected clusters), and
 * (optional) q_rot [L, G, 128] = rotate(q, cache_len) / sqrt(d) (fp32, fp64 angles) and the
 * contiguous-centroid list rej_w [L, rej_cap, GP] = logit + ln N of every centroid with the
 * selected ones -inf (replacement != 0) -- the inputs of mpa_sparse_decode.
 * k_new / v_new (fp32 [L, 128], optional): the step's key / value written at row cache_len after the
 * lists were cut, then the last CTA advances cache_len[s] and ntok_dense[l] (optional) by one
 * (ticket: one int32 workspace, zero-initialised once, left zeroed).
 * n_max bounds every ledger's cluster count (0: cap). */
/* 1 if mpa_decode_step can run n_ledgers ledgers of up to n_max centroids on the current device
 * (one co-resident wave of clusters, each CTA's slice within its shared-memory schedule), else 0 --
 * callers then take the staged kernels (mpa_centroid_logits + mpa_select_worklist). */
int mpa_decode_step_fits(int n_ledgers, int group, int n_max);

int mpa_decode_step(const float* q, const float* k_new, const float* v_new, const mpa_cache* cache,
                    const double* cs_lk, const double* inv_freq, int n_kv_heads, int group,
                    const mpa_level* fine, const int64_t* budget, const int32_t* sink_end,
                    const int32_t* buffer_start, int32_t* cache_len, int32_t* ntok_dense,
                    int32_t* ticket, int replacement, uint8_t* flag, int32_t* sel_tokens, int32_t* tok,
                    int tok_cap, int32_t* stats, int n_max, float* q_rot, float* rej_w, int rej_cap,
                    void* stream);


/* Work lists for the fused kernel (attention.py:469-496):
 *   tok[l, :]  = sinks [0, min(sink_end, cache_len)) ++ buffer [buffer_start, cache_len)
 *                ++ members of selected fine candidates;  n_tok[l]
 *   rej[l, :]  = rejected centroids as value-row codes (>= 0 fine row, < 0: coarse row -1-code)
 *                with rej_w[l, j, g] = logit + ln(size) (fp32, row stride GP = G <= 4 ? 4 : 8
 *                floats so a 16-row tile of logits is one aligned bulk copy);  n_rej[l]
 * Fine candidates: (cand, n_cand, flag, logits); coarse rejected (hier only, may be NULL):
 * (clogits, cflag) over the coarse level.  replacement == 0 drops every centroid term
 * ("flat-no-replacement", attention.py:441).  stats is [4, L]: rows n_tok, n_rej, sel_tokens,
 * n_selected_clusters (rows 0 and 1 feed mpa_sparse_decode directly).  sink_end / buffer_start / cache_len are per sequence [n_seq].
 *
 * K10 + work list fused in one launch per ledger: mpa_select over the fine candidates (extras =
 * coarse clusters with cflag == 0, hierarchy only) followed by the work lists above.
 * rej == NULL with replacement (flat level only): contiguous-centroid work list -- no rejected
 * list is written; rej_w already holds every candidate's weight (mpa_centroid_logits rej_w) and
 * the selected candidates' rows are set to -inf, so mpa_sparse_decode can stream the fine value
 * centroids [0, count[l]) in order (see there).  stats row 1 still counts the rejected; e_local
 * is consumed (its L2 lines are discarded without write-back: undefined afterwards). */
int mpa_select_worklist(const mpa_level* fine, const mpa_level* coarse, int group, const double* logits,
                        const double* e_local, const int32_t* cand, const int32_t* n_cand, int cand_cap,
                        const double* chunk_stats,
                        const uint8_t* cflag, const double* clogits, const int64_t* budget,
                        const int32_t* sink_end, const int32_t* buffer_start, const int32_t* cache_len,
                        int n_kv_heads, int n_ledgers, int replacement, uint8_t* flag,
                        int32_t* sel_tokens, int32_t* tok, int tok_cap, int32_t* rej, float* rej_w,
                        int rej_cap, int32_t* stats, int n_max, void* stream);

/* K11 + K12 -- fused sparse decode: one online softmax over the exact tokens (K_rot/V gathered
 * by index, logits q_rot . k) and the rejected-centroid pseudo-tokens (logit + ln N, value
 * centroid), LSE-merged in-kernel by the last finisher of each ledger
 * (attention.py:58-87, 120-137, 210-239, 473-498).  tok == NULL: dense decode over
 * [0, n_tok[l]) (the "oracle" comparator, attention.py:90-102).  Centroid terms: rej != NULL:
 * the listed value rows; rej == NULL and rej_w != NULL (stream-K path only): every fine value
 * centroid [0, n_rej[l]) in order with rej_w indexed by centroid (-inf = selected, no term);
 * rej_w == NULL: none.  rej_w rows have stride
 * GP = G <= 4 ? 4 : 8 floats.  bf16 caches with d in {64, 128}: stream-K tensor-core kernel
 * whose grid is one full wave (n_split <= 0) or n_split CTAs per ledger (used to test that the
 * result does not depend on the partition); other caches: FFMA kernel with n_split (0: auto)
 * CTAs per ledger.  workspace: >= mpa_sparse_decode_workspace(...) bytes, zero-filled once
 * before first use (the kernel leaves its ticket area zeroed).  out: fp32 [n_seq, Hq, d]. */
size_t mpa_sparse_decode_workspace(int n_ledgers, int group, int head_dim, int dtype, int n_split);
int mpa_sparse_decode(const mpa_cache* cache, const float* q_rot, int n_kv_heads, int group,
                      const int32_t* tok, const int32_t* n_tok, int tok_cap,
                      const int32_t* rej, const float* rej_w, const int32_t* n_rej, int rej_cap,
                      const void* fine_vc, int fine_cap, const void* coarse_vc, int coarse_cap,
                      int n_split, void* workspace, size_t workspace_bytes, float* out, void* stream);

/* ------------------------------------------------------------------------------------------
 * Sequence-sharded decode (one long context over P ranks): rank r holds a
 * contiguous range of every ledger's W-blocks (the last rank also the final block, sinks and
 * buffer); fine ids are global = gid_off[l] + local id, so the reference's (block, cluster)
 * tie-break order is preserved.  Per step:
 *   1. mpa_centroid_logits (local) -> mpa_head_norms -> all-gather -> mpa_merge_norms: the
 *      global (M, Z) of Eq. 1 (attention.py:276-278 normalise over ALL clusters of the head);
 *   2. mpa_select_worklist_sharded(prefix): each rank's candidates that can be globally selected
 *      (its local take-while-cum<B prefix) -> all-gather -> mpa_global_cut: the global crossing
 *      candidate, identical on every rank (attention.py:192-207);
 *   3. mpa_select_worklist_sharded(cross): flags + work lists of the local candidates;
 *   4. mpa_sparse_decode_partials -> all-gather -> mpa_merge_rank_partials (attention.py:230-239).
 * Heads / batch shard without any exchange. */
typedef struct mpa_prefix_entry {
    uint64_t key;     /* ~bits(score): ascending key == descending score */
    uint32_t gid;     /* global cluster id */
    int32_t size;
} mpa_prefix_entry;
typedef struct mpa_cross {
    uint64_t key;     /* 0: select none; ~0: select all */
    uint32_t gid;
    uint32_t pad;
} mpa_cross;

/* out[l, g] = (M, Z) of this rank's candidates from mpa_centroid_logits' chunk partials. */
int mpa_head_norms(const double* chunk_stats, int n_chunks, const int32_t* count, int n_ledgers, int group,
                   double* out, void* stream);
/* parts [P, L, G, 2] (every rank's (M, Z)) -> out [L, G, 2] global (M, Z). */
int mpa_merge_norms(const double* parts, int n_ranks, int n_ledgers, int group, double* out, void* stream);
/* Flat selection of a sharded ledger with the global normalisers mz [L, G, 2] and global ids
 * gid_off[l] + i.  Local pass (prefix != NULL, cross == NULL): writes the rank's candidate prefix
 * prefix[l, 0 .. prefix_n[l]) (prefix_n zeroed by the caller, capacity prefix_cap >= budget + 1).
 * Final pass (cross != NULL): flags, sel_tokens, work lists and stats as mpa_select_worklist. */
int mpa_select_worklist_sharded(const mpa_level* fine, int group, const double* logits, const double* e_local,
                                const double* chunk_stats, const int64_t* budget, const int32_t* sink_end,
                                const int32_t* buffer_start, const int32_t* cache_len, int n_kv_heads,
                                int replacement, uint8_t* flag, int32_t* sel_tokens, int32_t* tok, int tok_cap,
                                int32_t* rej, float* rej_w, int rej_cap, int32_t* stats, int n_max,
                                const double* mz, const void* cross, void* prefix, int32_t* prefix_n,
                                int prefix_cap, const int32_t* gid_off, void* stream);
/* prefix [P, L, cap] + prefix_n [P, L] of every rank -> cross [L] (mpa_cross). */
int mpa_global_cut(const void* prefix, const int32_t* prefix_n, int n_ranks, int n_ledgers, int prefix_cap,
                   const int64_t* budget, void* cross, void* stream);
/* mpa_sparse_decode writing per (ledger, q-head) partials [L, G, 2 + d] = (m natural-log, s,
 * a[d]) instead of a / s. */
int mpa_sparse_decode_partials(const mpa_cache* cache, const float* q_rot, int n_kv_heads, int group,
                               const int32_t* tok, const int32_t* n_tok, int tok_cap,
                               const int32_t* rej, const float* rej_w, const int32_t* n_rej, int rej_cap,
                               const void* fine_vc, int fine_cap, const void* coarse_vc, int coarse_cap,
                               int n_split, void* workspace, size_t workspace_bytes, float* part_out,
                               void* stream);
/* parts [P, L, G, 2 + d] -> out [L, G, d] (LSE merge + finalize). */
int mpa_merge_rank_partials(const float* parts, int n_ranks, int n_ledgers, int group, int head_dim, float* out,
                            void* stream);

/* ------------------------------------------------------------------------------------------
 * Clustering (K2-K8).  A batch of independent k-means "problems" p, each over a contiguous run
 * of points: rows prob_start[p] .. +prob_n[p] of ledger prob_l[p] -- either pre-rotation keys
 * (pts: [L, tcap, d] in pts_dtype) or fp64 rows (pts64: [L, rows64_cap, d], the fine centroids,
 * with integer weights wts [L, rows64_cap] for the hierarchy's size-weighted k-means).
 * Per-point arrays are indexed pt_off[p] + i, per-centroid arrays c_off[p] + j.
 * (clustering.py:84-184 Lloyd, :210-264 hierarchy, :343-472 online update / split / settle.) */
typedef struct mpa_km {
    int32_t n_prob;
    int32_t d;
    const void* pts;
    int32_t pts_dtype;
    int32_t tcap;
    const double* pts64;
    const int32_t* wts;
    int32_t rows64_cap;
    int32_t n_max;           /* max prob_n (grid sizing) */
    int32_t k_max;           /* max prob_k */
    int32_t min_iters;       /* Lloyd minimum update rounds (clustering.py:123-143) */
    const int32_t* prob_l;
    const int32_t* prob_start;
    const int32_t* prob_n;
    const int32_t* prob_k;
    const int32_t* pt_off;
    const int32_t* c_off;
    int32_t* assign;         /* [sum n] current assignment                 */
    int32_t* prev;           /* [sum n] previous round's assignment         */
    double* p2;              /* [sum n] squared point norms                 */
    double* cent;            /* [sum k, d] fp64 centroids (in: init; out: final) */
    double* c2;              /* [sum k]                                      */
    int32_t* count;          /* [sum k]                                      */
    int32_t* order;          /* [sum n] point ids grouped by cluster, ascending within */
    int32_t* cstart;         /* [sum k] first position of each cluster in order */
    int32_t* state;          /* [n_prob, 4] active, rounds, changed, has_empty */
    int32_t* flag;           /* [2] device scratch for the Lloyd driver loop (any active, max rounds) */
    /* tensor-core assignment (bf16 points, d = 128): optional; NULL -> fp64 CUDA-core kernel */
    int64_t pts_rows;        /* rows of the pts source ([L, tcap] flattened)            */
    int32_t sum_n, sum_k;    /* total points / centroids of the batch                    */
    void* tc_ws;             /* >= mpa_km_tc_workspace(n_prob, sum_k, sum_n, d) bytes    */
    int64_t tc_ws_bytes;
    int32_t* dirty;          /* [sum k] optional scratch: clusters whose members changed in the last
                                round (NULL: every centroid is recomputed every round)          */
} mpa_km;

/* Workspace of the tcgen05 assignment path (bf16 centroid terms, norms, recheck list). */
size_t mpa_km_tc_workspace(int n_prob, int sum_k, int sum_n, int d);

/* Lloyd to a fixed point for every problem (assign -> repair empties -> converged? -> means),
 * at least min_iters update rounds and at most min_iters + 100 (clustering.py:30, 123-143).
 * The assignment is the fp64 argmin of ||p||^2 + ||c||^2 - 2 p.c (first minimum) -- with
 * tc_ws given (bf16 points, d = 128) the contraction runs on tcgen05 with fp64 certification of
 * every point's best-vs-second margin and an exact fp64 re-score of the rest; means are
 * sequential fp64 member sums in ascending point order (bit-equal to np.add.at / np.mean).
 * Weighted mode (wts != NULL) keeps the centroid of an empty cluster (clustering.py:236-242).
 * Host-driven loop: one 8-byte readback per round.  *rounds_out = max rounds over problems. */
int mpa_km_lloyd(const mpa_km* km, int32_t* rounds_out, void* stream);

/* Means / counts / grouping for the assignment already in km->assign (no iteration): used to
 * seed the two sides of a sliding-window split (clustering.py:368-383). */
int mpa_km_means(const mpa_km* km, void* stream);

/* nk[p] = number of non-empty clusters of problem p after Lloyd. */
int mpa_km_count_nonempty(const mpa_km* km, int32_t* nk, void* stream);

/* Compaction into a ledger level (clustering.py:146-167, 187-192): non-empty clusters of problem
 * p, in centroid order, become clusters f0[p] .. f0[p]+nk[p]-1 of ledger prob_l[p]:
 *   kc64 = centroid, vc64 = sequential mean of the members' value rows (vals: [L, tcap, d] in
 *   pts_dtype; NULL for the hierarchy), serving copies kc / vc in the cache dtype, size,
 *   CSR off[f0 + j] = mbase[p] + prefix, idx[mbase[p] + ...] = member ids (token ids
 *   prob_start + i for key problems, fine ids for the hierarchy -- "children").
 * Hierarchy (pts64 != NULL): kc64 / vc64 are the size-weighted means of the children's fine
 * centroids (fine_vc64 supplies the value side) -- clustering.py:249-255. */
int mpa_km_write_level(const mpa_km* km, const mpa_cache* vcache, const double* fine_vc64,
                       const int32_t* f0, const int32_t* mbase,
                       double* kc64, double* vc64, void* kc, void* vc, int32_t serve_dtype,
                       int32_t* size, int32_t* off, int32_t* idx, int32_t level_cap, int32_t idx_cap,
                       void* stream);

/* Initial assignment of a problem from an existing ledger level: point i (token prob_start + i)
 * gets the LOCAL id (cluster - first[p]) of the cluster of ledger prob_l[p] containing it
 * (first[p] .. first[p] + nclus[p] - 1 are searched).  Used by splits and settles. */
int mpa_km_assign_from_level(const mpa_km* km, const int32_t* off, const int32_t* idx, int32_t level_cap,
                             int32_t idx_cap, const int32_t* first, const int32_t* nclus,
                             const int32_t* mbase, void* stream);

/* K6 -- single-pass sequential assignment of the L appended tokens with running-mean updates
 * (clustering.py:439-444): for t in order: c = argmin_j ||cent_j - x_t||^2 (direct form, first
 * min); count[c] += 1; cent[c] += (x_t - cent[c]) / count[c].  One CTA per ledger; cent / count
 * are per-problem arrays at c_off[p] with k = prob_k[p]; tokens prob_start[p] + tail_start[p] ..
 * +n_new.  dist is [n_prob, n_new, k_max] fp64 workspace. */
int mpa_km_seq_assign(const mpa_km* km, const int32_t* tail_start, int n_new, double* dist, void* stream);


/* ---- fp64 kernels behind the reference's module-level Python API (attention.*, rope.*,
 * clustering.* for numpy / Cluster / BlockLedger callers; paper_2506_13059_b200/{attention,rope,
 * clustering}.py).  Device pointers, one stream, row-major fp64 unless noted. */
/* rope.py:37-53 `rotate`: out[r] = x[r] rotated by pos[r] * inv_freq (fp64 positions, interleaved pairs). */
int mpa_ref_rotate(const double* x, const double* pos, int n, int d, const double* inv_freq, double* out,
                   void* stream);
/* attention.py:84-86, 154, 276: out[g, j] = q[g] . x[j] / sqrt(d). */
int mpa_ref_logits(const double* q, const double* x, int G, int n, int d, double* out, void* stream);
/* attention.py:58-68 `_partial_from_logits`: m = max l, w = exp(l - m) * weights (NULL: 1), s = sum w,
 * a = w @ values; out = [a (d), m, s]; weights_out (optional) = w / s (attention.py:105-117). */
int mpa_ref_partial(const double* logits, const double* values, const double* weights, int n, int d,
                    double* out, double* weights_out, void* stream);
/* attention.py:144-164, 267-290: scores[j] = mean_g e[g, j] / (e[g] . sizes), e = exp(l - max_g);
 * z_out (optional) [G] = the normalisers. */
int mpa_ref_group_scores(const double* logits, const double* sizes, int G, int n, double* scores,
                         double* z_out, void* stream);
/* clustering.py:84-88 + argmin: assign[i] = first minimum of |p|^2 + |c|^2 - 2 p . c. */
int mpa_ref_nearest(const double* points, const double* centroids, int n, int k, int d, int64_t* assign,
                    void* stream);
/* clustering.py:113-120, 195-203, 255-257: per cluster c (CSR off[k + 1] / idx into the rows of
 * points): mean[c] = in-order sum / count, or with weights (per point row) sum w x / sum w (optional);
 * with centroids, *sqerr += sum |p - centroids[c]|^2. */
int mpa_ref_seg_stats(const double* points, const int64_t* off, const int64_t* idx, const double* weights,
                      int k, int d, double* mean, const double* centroids, double* sqerr, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MPATTN_H */
