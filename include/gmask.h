/*
 * gmask.h — C ABI of libgmask.so, the B200-native token-mask engine.
 *
 * This is the drop-in boundary for the reference's token-mask hot path
 * (grammask, /root/reference/pkg/src/grammask).  Every entry point names the
 * reference interface it replaces (REF = /root/reference/pkg/src/grammask).
 * The Python host layer (paper_2411_15100_b200/_lib.py) binds these with
 * ctypes; INTEGRATION.md shows the binding a maintainer of the reference
 * would add.
 *
 * Conventions
 *   - plain C types only: pointers + sizes, no torch types.
 *   - "device pointer" arguments are CUDA global-memory addresses owned by
 *     the caller (torch tensors in the Python layer); "host pointer"
 *     arguments are ordinary host memory.
 *   - all kernel launches are stream-ordered on the given cudaStream_t
 *     (passed as void* so the header needs no CUDA include); 0 = legacy
 *     default stream.  No call on the per-step path allocates memory or
 *     synchronises the stream, except where documented ("syncs").
 *   - every function returns gm_status; on failure gm_last_error() returns a
 *     thread-local message.
 *   - handles (gm_vocab, gm_grammar, gm_cache, gm_pool) are library-owned and
 *     released with the matching *_release.
 */
#ifndef GMASK_H_
#define GMASK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t gm_status;
enum {
  GM_OK = 0,
  GM_ERR_INVALID = 1,     /* bad argument (MatcherError/ValueError in Python)   */
  GM_ERR_CUDA = 2,        /* CUDA runtime failure                               */
  GM_ERR_STATE_CAP = 3,   /* stack/branch set exceeded its cap (REF pda.py:53-57,
                             cache.py:137-138, matcher.py:188-189)               */
  GM_ERR_TERMINATED = 4,  /* matcher terminated (REF matcher.py:251-252, 379-381) */
  GM_ERR_SHAPE = 5,       /* mask/bitmask shape mismatch (REF matcher.py:382-383) */
  GM_ERR_ARENA_FULL = 6,  /* device stack arena exhausted                        */
  GM_ERR_ROLLBACK = 7,    /* rollback beyond history (REF matcher.py:313-314)    */
  GM_ERR_OOM = 8,
  GM_ERR_GRAMMAR = 9      /* grammar outside the engine's limits (GrammarError) */
};

/* Thread-local description of the last failure on this thread. */
const char* gm_last_error(void);
const char* gm_version(void);

/* ------------------------------------------------------------------------ */
/* K0: apply_token_bitmask_inplace                                           */
/* ------------------------------------------------------------------------ */
/* Replaces XGrammar's apply_token_bitmask_inplace
 * (xgrammar/matcher.py:58-188; absent in the reference — grammask never
 * touches logits, REF bench.py:50-71).  For every row r (r = indices[i] when
 * indices != NULL, else r = i for i < n_rows) and every token j < vocab_size:
 *     bit j of bitmask[r] == 0  =>  logits[r, j] = -inf
 * allowed logits are left bit-identical.  dtype: GM_DTYPE_*.  logits and
 * bitmask are device pointers; strides are in elements. */
enum { GM_DTYPE_F32 = 0, GM_DTYPE_F16 = 1, GM_DTYPE_BF16 = 2 };
gm_status gm_apply_inplace(void* logits, int32_t dtype, int64_t n_rows,
                           int64_t vocab_size, int64_t logits_stride,
                           const int32_t* bitmask, int64_t bitmask_stride,
                           const int32_t* indices, void* stream);

/* K0's policy for 16-byte chunks that mix allowed and masked logits: a
 * warp whose store round has at least min_lanes mixed chunks loads them,
 * blends in -inf and writes each with one full store; otherwise (or with
 * min_lanes = 0) it writes only the masked elements.  Returns the previous
 * value.  Default: GMASK_APPLY_BLEND at load, else the build's default.
 * The fused apply (K3/K5) blends the rows of the cache keys whose accepted
 * row meets the same thresholds (scaled to the row), decided when the cache
 * is built (gm_cache_create) with the policy in force then. */
int32_t gm_apply_set_blend(int32_t min_lanes);

/* ------------------------------------------------------------------------ */
/* Vocabulary                                                                */
/* ------------------------------------------------------------------------ */
/* Replaces Vocabulary + SortedVocabIndex (REF vocab.py:111-134, 203-234).
 * bytes/offsets are host pointers: token i = bytes[offsets[i]:offsets[i+1]].
 * special must contain eos_id (REF vocab.py:141).  The library uploads the
 * token bytes, the lexicographic order of non-special non-empty tokens
 * (ties by id, REF vocab.py:227-234) and the universe bitset (non-special,
 * non-empty tokens, REF matcher.py:141-144) to the current device. */
typedef struct gm_vocab gm_vocab;
gm_status gm_vocab_create(const uint8_t* bytes, const int64_t* offsets,
                          int32_t vocab_size, const int32_t* special,
                          int32_t n_special, int32_t eos_id, gm_vocab** out);
void gm_vocab_release(gm_vocab* v);
int32_t gm_vocab_size(const gm_vocab* v);
/* Device pointer to the universe row (ceil(V/32) int32 words). */
const int32_t* gm_vocab_universe(const gm_vocab* v);

/* ------------------------------------------------------------------------ */
/* Grammar tables (output of the host front end)                             */
/* ------------------------------------------------------------------------ */
/* The front end (paper_2411_15100_b200/automaton.py) lowers grammar text to a
 * byte-level pushdown automaton whose silent moves (epsilon, rule push,
 * frame-internal pop) are pre-closed into per-(node, byte-class) transition
 * lists.  A transition (target, push run) means: push the return nodes
 * push_pool[off .. off+len) in order, then rest on `target`.
 * node_flags: GM_NODE_POP   = node can silently complete its rule (pop the
 *                             frame), the SC(n) fact of SURVEY §7;
 *             GM_NODE_DEAD_END = final node with no moves except the pop
 *                             (REF pda.py:131-134).
 * follow_* is the context-expansion automaton (REF cache.py:241-333) as a
 * DFA over byte classes: state -1 = dead, -2 = wildcard (anything follows). */
enum { GM_NODE_POP = 1, GM_NODE_DEAD_END = 2 };
enum { GM_FOLLOW_DEAD = -1, GM_FOLLOW_ANY = -2 };
typedef struct gm_grammar_tables {
  int32_t n_nodes;
  int32_t n_rules;
  int32_t n_classes;
  int32_t start_node;          /* root rule start                              */
  const uint8_t* byte_class;   /* [256]                                        */
  const int32_t* trans_off;    /* [n_nodes*n_classes + 1] CSR offsets          */
  const int32_t* trans;        /* [2*n_trans]: target, push_off | push_len<<24 */
  int32_t n_trans;
  const int32_t* push_pool;    /* [n_push] return nodes                        */
  int32_t n_push;
  const uint8_t* node_flags;   /* [n_nodes]                                    */
  const int32_t* node_rule;    /* [n_nodes]                                    */
  const int32_t* cache_keys;   /* [n_keys] resting nodes (cache key set),
                                  REF pda.py:601-632                           */
  int32_t n_keys;
  const int32_t* follow_start; /* [n_rules]                                    */
  const int32_t* follow_next;  /* [n_fstates*n_classes]                        */
  int32_t n_fstates;
} gm_grammar_tables;

/* ------------------------------------------------------------------------ */
/* Native host front end                                  */
/* ------------------------------------------------------------------------ */
/* Replaces the reference's PDA construction and optimisation passes and the
 * FollowFsa precompute (REF pda.py:246-535, cache.py:241-333) with the
 * automaton construction of paper_2411_15100_b200/automaton.py in C++: per
 * rule subset construction + Moore minimisation, inlining of small call-free
 * rules, silent-move pre-closure, follow DFA.  Input: the parsed grammar as
 * an int32 prefix IR (front_end.cpp header), n_rules bodies in rule-id order.
 * Output: tables in the gm_grammar_tables layout (kept_rules[i] = source rule
 * id of device rule i), owned by the returned handle.  Host only (no GPU).
 * Errors: GM_ERR_STATE_CAP (closure cap, REF pda.py:53-57), GM_ERR_GRAMMAR. */
typedef struct gm_fe_options {
  int32_t determinize;              /* must be 1 (CompileOptions.merge)      */
  int32_t inline_rules;             /* CompileOptions.inline                 */
  int32_t ctx_expansion;            /* CompileOptions.ctx_expansion          */
  int32_t inline_max_rule_states;   /* 32                                    */
  int32_t inline_max_result_states; /* 1024                                  */
  int32_t max_dfa_states;           /* 200000                                */
  int32_t max_follow_states;        /* 4096                                  */
  int32_t state_cap;                /* 4096 (REF pda.py:53)                  */
  int32_t inline_calls;             /* 1: also inline single-caller rules    */
} gm_fe_options;

typedef struct gm_fe_tables {
  int32_t n_nodes, n_rules, n_classes, start_node, root_rule;
  int32_t n_trans, n_push, n_keys, n_fstates;
  const uint8_t* byte_class;
  const int32_t* trans_off;
  const int32_t* trans;
  const int32_t* push_pool;
  const uint8_t* node_flags;
  const int32_t* node_rule;
  const int32_t* cache_keys;
  const int32_t* follow_start;
  const int32_t* follow_next;
  const int32_t* kept_rules;
  /* the per-rule DFAs before the pre-closure (for bundle export): node u's
   * edges raw[2*raw_off[u] .. 2*raw_off[u+1]) as (symbol, dst), symbol >= 0
   * a byte class, < 0 a call of rule -(symbol+1) returning to dst */
  const int32_t* raw_off;      /* [n_nodes + 1] */
  const int32_t* raw;          /* [2 * n_raw]   */
  int32_t n_raw;
  const uint8_t* finals;       /* [n_nodes]     */
  const int32_t* rule_start;   /* [n_rules]     */
} gm_fe_tables;

/* Native grammar parser (the rest of SURVEY §8f rank 2): EBNF text (UTF-8,
 * len bytes) -> the prefix IR gm_front_end_build takes, with the rule names
 * ('\0'-separated, name i = names + name_off[i]) and the root rule index
 * (root_rule_name, nullable: `root` if defined, else the first rule).
 * Surface semantics and every error message / position are those of REF
 * grammar.py (restated in paper_2411_15100_b200/grammar.py, which the tests
 * compare it with).  On GM_ERR_GRAMMAR the view's error / err_line /
 * err_col describe the GrammarError (line 0: no position) and *out must
 * still be released.  Host only. */
typedef struct gm_parsed gm_parsed;
typedef struct gm_parse_view {
  const int32_t* ir;
  int64_t ir_len;
  int32_t n_rules;
  int32_t root_rule;
  const char* names;
  const int64_t* name_off;   /* [n_rules + 1] */
  const char* error;
  int32_t err_line, err_col;
} gm_parse_view;
gm_status gm_grammar_parse(const uint8_t* text, int64_t len, const char* root_rule_name,
                           gm_parsed** out, gm_parse_view* view);
void gm_grammar_parse_release(gm_parsed* g);

typedef struct gm_front_end gm_front_end;
gm_status gm_front_end_build(const int32_t* ir, int64_t ir_len, int32_t n_rules,
                             int32_t root_rule, const gm_fe_options* opts,
                             gm_front_end** out, gm_fe_tables* view);
void gm_front_end_release(gm_front_end* fe);

typedef struct gm_grammar gm_grammar;
/* Copies the (host) tables to the current device. */
gm_status gm_grammar_create(const gm_grammar_tables* t, gm_grammar** out);
void gm_grammar_release(gm_grammar* g);

/* ------------------------------------------------------------------------ */
/* K1/K1b: adaptive token-mask cache build                                   */
/* ------------------------------------------------------------------------ */
/* Replaces build_mask_cache / sweep / FollowFsa refinement
 * (REF cache.py:88-193, 241-333, 516-574).  For each key index k in
 * [key_begin, key_begin+n) (into tables.cache_keys) and every non-special,
 * non-empty token t, classifies t from a synthetic single-frame stack at the
 * key node: accepted (bit set in acc_rows[k-key_begin]), context dependent
 * after context expansion (bit set in dep_rows[k-key_begin]) or rejected
 * (neither bit).  acc_rows/dep_rows are device [n x ceil(V/32)] int32,
 * zero-filled by this call.  Position sharding across GPUs = disjoint
 * [key_begin, key_begin+n) ranges, then an all-gather of the rows. */
gm_status gm_cache_build_rows(const gm_grammar* g, const gm_vocab* v,
                              int32_t key_begin, int32_t n,
                              int32_t* acc_rows, int32_t* dep_rows,
                              void* stream);

/* Position sharding with any subset of keys: rows of the keys listed in the
 * HOST array key_list[0..n) (indices into tables.cache_keys, any order; row
 * i of acc_rows/dep_rows belongs to key_list[i]).  The Python layer deals
 * the keys of a build round-robin in decreasing order of estimated walk
 * cost and replicates the rows with one all-gather issued
 * through torch.distributed (ProcessGroupNCCL over NVLink): the library
 * takes no NCCL dependency, the payload is one contiguous device buffer per
 * rank either way.  Syncs the stream. */
gm_status gm_cache_build_keys(const gm_grammar* g, const gm_vocab* v,
                              const int32_t* key_list, int32_t n,
                              int32_t* acc_rows, int32_t* dep_rows,
                              void* stream);
int32_t gm_grammar_num_keys(const gm_grammar* g);

/* Assemble a cache from complete rows for all keys (device pointers; the
 * rows are copied).  Dependent bit rows are compacted to sorted id lists
 * (REF cache.py:400-402).  Syncs the stream. */
typedef struct gm_cache gm_cache;
typedef struct gm_cache_stats {
  int32_t n_keys;
  int64_t accepted_total;   /* REF cache.py:423-437 BuildStats */
  int64_t dependent_total;
  int64_t rejected_total;
  int64_t row_bytes;        /* dense rows resident in HBM */
  int32_t blend_keys;       /* keys whose rows the fused apply blends (gm_apply_set_blend) */
} gm_cache_stats;
gm_status gm_cache_create(const gm_grammar* g, const gm_vocab* v,
                          const int32_t* acc_rows, const int32_t* dep_rows,
                          gm_cache** out, gm_cache_stats* stats, void* stream);
void gm_cache_release(gm_cache* c);
/* Export for inspection / GMC1 serialisation: copies the accepted rows
 * [n_keys x W], dependent offsets [n_keys+1] and dependent ids [n_dep] into
 * caller device buffers (each nullable).  Syncs. */
gm_status gm_cache_export(const gm_cache* c, int32_t* acc_rows_out, int32_t* dep_off_out,
                          int32_t* dep_ids_out, int64_t* n_dep_out);

/* ------------------------------------------------------------------------ */
/* Matcher pool: device-resident persistent stacks                           */
/* ------------------------------------------------------------------------ */
/* Replaces Matcher state + StackArena (REF matcher.py:103-154, 239-355,
 * pstack.py:24-111).  A pool holds `capacity` matcher slots.  Every slot
 * keeps a ring of (history_window+1) stack-top sets of at most max_stacks
 * (handle, node) pairs; handles index a device hash-consed arena of
 * (parent, return-node) frames shared by all slots (equal content => equal
 * handle, so branch/rollback cost one handle copy per stack). */
typedef struct gm_pool gm_pool;
gm_status gm_pool_create(int32_t capacity, int32_t max_stacks,
                         int32_t max_window, int64_t arena_log2,
                         gm_pool** out);
void gm_pool_release(gm_pool* p);

/* Bind slot to (grammar, cache, vocab) and reset it to the start state
 * (REF matcher.py:154).  window = rollback history length for this slot. */
gm_status gm_pool_reset(gm_pool* p, int32_t slot, const gm_grammar* g,
                        const gm_cache* c, const gm_vocab* v, int32_t window,
                        void* stream);
/* Copy slot src to dst, history included (REF matcher.py:328-355 branch). */
gm_status gm_pool_fork(gm_pool* p, int32_t src, int32_t dst, void* stream);

/* K4: batched accept_token.  slots/token_ids are device int32[n];
 * accepted_out device uint8[n] (1 = accepted).  Semantics of REF
 * matcher.py:273-294: EOS terminates iff terminable; special or empty
 * tokens are rejected; a rejected token leaves the slot unchanged. */
gm_status gm_accept_tokens(gm_pool* p, const int32_t* slots,
                           const int32_t* token_ids, int32_t n,
                           uint8_t* accepted_out, void* stream);
/* accept_bytes / accept_string for one slot (REF matcher.py:248-271);
 * data is a host pointer; the result is written to accepted_out (device). */
gm_status gm_accept_bytes(gm_pool* p, int32_t slot, const uint8_t* data,
                          int64_t len, uint8_t* accepted_out, void* stream);

/* K2: batched fill_next_token_bitmask.  For i < n: row = rows ? rows[i] : i,
 * bitmask[row] (device, int32, row stride bitmask_stride) receives the
 * permitted-token mask of slots[i] (REF matcher.py:377-444): universe AND
 * union over stacks of (cached accepted row OR walked dependents), EOS bit
 * iff terminable, bits >= V zero.  need_apply_out[i] (nullable, device
 * uint8) = mask is not all-ones over the vocabulary. */
gm_status gm_fill_tokens(gm_pool* p, const int32_t* slots, int32_t n,
                         int32_t* bitmask, int64_t bitmask_stride,
                         const int32_t* rows, uint8_t* need_apply_out,
                         void* stream);

/* K3: fused fill + apply.  For i < n (row = rows ? rows[i] : i) computes the
 * mask of slots[i] exactly as gm_fill_tokens, optionally stores it to
 * bitmask[row] (bitmask nullable), and masks logits[row, :vocab_size] in
 * place exactly as gm_apply_inplace — one launch, no bitmask round trip
 * through HBM.  dtype: GM_DTYPE_*; logits rows must be 16-byte aligned. */
gm_status gm_fill_apply_tokens(gm_pool* p, const int32_t* slots, int32_t n,
                               int32_t* bitmask, int64_t bitmask_stride,
                               const int32_t* rows, void* logits, int32_t dtype,
                               int64_t vocab_size, int64_t logits_stride,
                               void* stream);

/* K5: one decode step per request — accept, then fill (+ apply).  For
 * i < n: if token_ids is non-null, accept token_ids[i] on slots[i] exactly as
 * gm_accept_tokens (accepted_out[i] = 1/0; a rejected token leaves the state
 * unchanged); with recycle_terminated != 0 a request that terminates is
 * restarted at the grammar's start state (gm_pool_recycle); then fill the
 * slot's next mask exactly as gm_fill_tokens into bitmask[row] (nullable when
 * logits is given) and, when logits is non-null, apply it to logits[row] as
 * gm_fill_apply_tokens.  A request that terminated in this step (and is not
 * recycled) gets an all-zero row and no error.  Replaces the accept_token ->
 * fill_next_token_bitmask pair of a decode loop (REF matcher.py:273, 377)
 * with one launch. */
gm_status gm_step_tokens(gm_pool* p, const int32_t* slots, int32_t n,
                         const int32_t* token_ids, uint8_t* accepted_out,
                         int32_t recycle_terminated, int32_t* bitmask,
                         int64_t bitmask_stride, const int32_t* rows,
                         void* logits, int32_t dtype, int64_t vocab_size,
                         int64_t logits_stride, void* stream);

/* gm_step_tokens with the slot ids passed by value from HOST memory
 * (host_slots[0..n), n <= 512, rows = i): the step kernel's first global
 * access is then the slot header itself, one round trip fewer.  Token ids
 * (device, nullable: first step), outputs and semantics as gm_step_tokens. */
gm_status gm_step_tokens_host_slots(gm_pool* p, const int32_t* host_slots, int32_t n,
                                    const int32_t* token_ids, uint8_t* accepted_out,
                                    int32_t recycle_terminated, int32_t* bitmask,
                                    int64_t bitmask_stride, void* logits, int32_t dtype,
                                    int64_t vocab_size, int64_t logits_stride,
                                    void* stream);

/* Native decode loop over gm_step_tokens with host buffers (the serving
 * form of the reference's per-token accept_token -> fill_next_token_mask
 * loop, REF matcher.py:273, 377, driven from the host as in REF bench.py:
 * 287-338).  A decoder owns n_buf step slots; slot b has pinned host staging
 * for the token ids and accepted flags, device copies, and its bitmask /
 * logits buffers (device pointers, caller-owned; bitmasks may be NULL).
 * gm_decoder_step(d, b, host_tokens, stream) issues one decode step without
 * blocking: waits (host) until slot b's previous step has completed, copies
 * host_tokens (int32[n], NULL = first step: fill + apply only) into slot b's
 * staging, then H2D copy on the decoder's copy stream -> K5 (accept +
 * recycle + fill + apply) on `stream` -> D2H copy of the accepted flags,
 * ordered by events so the copies of neighbouring steps overlap the
 * kernels.  gm_decoder_flags(d, b, out, wait) copies slot b's latest
 * accepted flags (uint8[n]) to host memory `out` (wait = 1: block until
 * that step completed; 0: caller already waited), returning GM_ERR_INVALID
 * when the step has not completed and wait = 0. */
typedef struct gm_decoder gm_decoder;
gm_status gm_decoder_create(gm_pool* p, const int32_t* slots, int32_t n,
                            int32_t n_buf, int32_t* const* bitmasks,
                            int64_t bitmask_stride, void* const* logits,
                            int32_t dtype, int64_t vocab_size,
                            int64_t logits_stride, int32_t recycle,
                            gm_decoder** out);
gm_status gm_decoder_step(gm_decoder* d, int32_t buf,
                          const int32_t* host_tokens, void* stream);
gm_status gm_decoder_flags(gm_decoder* d, int32_t buf, uint8_t* out,
                           int32_t wait);
void gm_decoder_release(gm_decoder* d);

/* rollback `steps` acceptances of each slot (REF matcher.py:310-326);
 * slots/steps are device int32[n]. */
gm_status gm_rollback(gm_pool* p, const int32_t* slots, const int32_t* steps,
                      int32_t n, void* stream);

/* Serving-loop request recycling: every slot in slots[0..n) (device int32)
 * whose current state is terminated restarts at the grammar start with an
 * empty history; other slots are untouched.  Stream-ordered, no sync. */
gm_status gm_pool_recycle(gm_pool* p, const int32_t* slots, int32_t n, void* stream);

/* Introspection (syncs).  info = {n_stacks, terminated, history_len,
 * terminable, window}; stacks_out (nullable) receives up to max_out
 * (handle, node) pairs of the current top set. */
gm_status gm_pool_slot_info(gm_pool* p, int32_t slot, int32_t* info5,
                            int32_t* stacks_out, int32_t max_out);
/* Materialise a stack: frames bottom-up into out (host), returns depth via
 * *depth (REF pstack.py:70-77). */
gm_status gm_pool_materialize(gm_pool* p, int32_t handle, int32_t* out,
                              int32_t max_out, int32_t* depth);
/* Union of acceptable first bytes (256-bit, 8 words) and terminability over
 * the closure of the slot's current stacks (REF matcher.py:219-237); used
 * by jump-forward (REF matcher.py:464-486).  Syncs. */
gm_status gm_pool_first_bytes(gm_pool* p, int32_t slot, uint32_t* bytes8,
                              int32_t* terminable);
/* Sticky device error flags, OR over every slot of the pool (bit 1 << GM_ERR_*),
 * all cleared by the read.  Pool-wide diagnostic; per-request errors come
 * from gm_pool_errors.  Syncs. */
gm_status gm_pool_check(gm_pool* p, int32_t* flags_out);

/* Per-request errors.  A device error (stack set over the 4096 cap of REF
 * matcher.py:116/188-189, a terminated matcher stepped or filled, REF
 * matcher.py:276-277/379-381, arena exhaustion, a token id out of range) is
 * recorded in the error word of the slot whose operation failed, never
 * silently dropped: K4/K5 also return it in accepted_out (bit 1; bit 0 =
 * accepted) and the state is left unchanged.  gm_pool_errors gathers the
 * words of slots[0..n) (device int32) into out[0..n) (device uint32, bit
 * 1 << GM_ERR_*), clearing them when clear != 0.  Stream-ordered, no sync.
 * gm_status_of_error_bits maps a word to its gm_status (+ gm_last_error()
 * message), GM_OK for 0. */
gm_status gm_pool_errors(gm_pool* p, const int32_t* slots, int32_t n,
                         uint32_t* out, int32_t clear, void* stream);
gm_status gm_status_of_error_bits(uint32_t bits);
/* Arena statistics (syncs): live frames, tombstones, capacity (slots). */
gm_status gm_pool_arena_stats(gm_pool* p, int64_t* live, int64_t* tombstones,
                              int64_t* capacity);
/* live frames (gm_pool_arena_stats), -1 on error */
int64_t gm_pool_arena_used(gm_pool* p);
/* Reclaim arena frames (REF pstack.py:85-111 decref / end_log: frames no
 * live stack references are freed).  live_slots (HOST int32[n]) lists every
 * slot whose state must survive; every other slot's history is dropped.
 * Frames reachable from a top of a live slot's history-ring entries (the
 * rollback window) are kept; the rest become free again.  Handles never
 * move, so live state is untouched.  Stream-ordered: no step kernel on
 * this pool may run concurrently on another stream. */
gm_status gm_pool_collect(gm_pool* p, const int32_t* live_slots, int32_t n,
                          void* stream);
/* Diagnostics: phase timestamps (ns, %globaltimer) of CTA 0 of the last
 * accept (out[0..16)) and fill (out[16..32)) launches, then per-CTA
 * durations (fill: out[64 + 2i], accept: out[64 + 2*capacity + i]) when the
 * pool was created with GMASK_TRACE=1; GM_ERR_INVALID otherwise.  Syncs. */
gm_status gm_pool_trace(gm_pool* p, uint64_t* out, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* GMASK_H_ */
