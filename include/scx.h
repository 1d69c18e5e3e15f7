/*
 * scx.h -- C-ABI of libscx.so, the sm_100a kernels behind the
 * paper_2506_09226_b200 relational operators.
 *
 * The reference (`/root/reference/pkg/src/shufflecast`) is pure numpy and has
 * no FFI; each entry point below replaces the numpy body of the Python
 * operator named in its comment (file:line under /root/reference/pkg/src/
 * shufflecast).  The Python host layer (paper_2506_09226_b200/*.py) keeps the
 * reference's operator/plan API and binds these through ctypes
 * (INTEGRATION.md shows the binding a shufflecast maintainer would add).
 *
 * Conventions
 *   - Every pointer argument named *_dev / uint64 "ptr" fields is a DEVICE
 *     address (e.g. torch.Tensor.data_ptr()).  Host pointers are named *_host.
 *   - Every call is asynchronous on `stream` (a cudaStream_t, passed as
 *     void*; NULL = legacy default stream).  Nothing allocates: callers pass
 *     scratch sized by the matching *_workspace query.
 *   - Return 0 on success, a negative SCX_E* code on error; the message is in
 *     scx_last_error() (thread-local).  No C++ exception crosses the ABI.
 *   - No global mutable state: safe to call from one thread per device.
 */
#ifndef SCX_H
#define SCX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCX_ABI_VERSION 1

/* ---- error codes ------------------------------------------------------- */
#define SCX_OK            0
#define SCX_EINVAL       -1   /* bad argument / descriptor                  */
#define SCX_ECUDA        -2   /* CUDA runtime error (launch, memset, ...)   */
#define SCX_ECAPACITY    -3   /* caller-provided buffer too small           */
#define SCX_EUNSUPPORTED -4   /* shape outside what the kernels implement   */

/* ---- physical column types (narrowed HBM layout) ---------- */
#define SCX_I8   0
#define SCX_I16  1
#define SCX_I32  2
#define SCX_I64  3
#define SCX_U8   4
#define SCX_U16  5
#define SCX_F64  6
#define SCX_U32  7

/* ---- limits of one pipeline descriptor --------------------------------- */
#define SCX_MAX_BASE      12   /* scanned (TMA-staged) columns              */
#define SCX_MAX_SLOTS     32   /* base + probe-payload operand slots        */
#define SCX_MAX_ATOMS     40
#define SCX_MAX_SETWORDS  128  /* dictionary-set bitmaps, 32 codes / word   */
#define SCX_MAX_LUT       512  /* dictionary code -> string-rank tables     */
#define SCX_MAX_PROBES    8
#define SCX_MAX_POLYS     4    /* polynomial comparison atoms per pipeline  */
#define SCX_MAX_PAYLOAD   6
#define SCX_MAX_MEASURES  8
#define SCX_MAX_GKEYS     4
#define SCX_MAX_OUT       16
#define SCX_MAX_KEYS      4    /* key columns of a join / partition key     */

/* atom ops: one comparison evaluated per row */
#define SCX_ATOM_RANGE  0      /* lo <= v[slot] <= hi                         */
#define SCX_ATOM_SET    1      /* bit v[slot] of setwords[set_word..] is 1;
                                  lo = number of bitmap words of the set     */
#define SCX_ATOM_DIFF   2      /* lo <= v[slot] - v[slot2] <= hi              */
#define SCX_ATOM_POLY   3      /* lo <= polys[slot](row) <= hi: exact int64
                                  polynomial of slots (scx_measure form)      */

/* join kinds for a probe stage (relops.py:59-94) */
#define SCX_JOIN_SEMI   0
#define SCX_JOIN_ANTI   1
#define SCX_JOIN_INNER  2      /* build keys unique: 0/1 match per probe row  */
#define SCX_JOIN_LEFT   3      /* left outer, unique build keys: every probe
                                  row kept, payload = 0 when unmatched       */

/* key component transforms (scx_keyspec.xform, 8 bits per component) */
#define SCX_XFORM_NONE  0
#define SCX_XFORM_YEAR  1      /* civil year of a date32 (days since 1970)    */

/* lookup-table kinds */
#define SCX_HT_HASH     0      /* open addressing, linear probing: keys = u64
                                  slots[2*cap], slot h = {key, row} (16 B)    */
#define SCX_HT_DIRECT   1      /* dense key range: vals[packed key]           */
#define SCX_HT_BITMAP   2      /* semi/anti membership: bit [packed key] of
                                  the u32 words at vals, cap = key domain    */
#define SCX_HT_IDENTITY 3      /* build key column is lo, lo+1, ...: the
                                  packed key IS the build row (< cap rows),
                                  no table at all                            */

/* aggregate ops (relops.py:11, AGG_OPS) */
#define SCX_AGG_SUM     0
#define SCX_AGG_COUNT   1
#define SCX_AGG_MIN     2
#define SCX_AGG_MAX     3

/* pipeline sinks */
#define SCX_SINK_AGG_DENSE 0   /* small key domain: register/smem pre-agg    */
#define SCX_SINK_AGG_HASH  1   /* open-addressing group table, global atomics */
#define SCX_SINK_COMPACT   2   /* stable stream compaction (decoupled look-back) */
#define SCX_SINK_COUNT     3   /* selected-row count only                      */
#define SCX_SINK_BITMAP    4   /* set bit [gkey-packed key] of the u32 words at
                                  gkeys (domain gcap): a semi/anti-join build
                                  side straight from a filtered scan         */

#define SCX_EMPTY_KEY 0xFFFFFFFFFFFFFFFFull
#define SCX_NO_ROW    0xFFFFFFFFu

typedef struct scx_column {
  uint64_t ptr;     /* device address of element 0 (16-byte aligned) */
  int32_t dtype;    /* SCX_I8 ... */
  int32_t _pad;
} scx_column;

typedef struct scx_atom {
  int32_t op;       /* SCX_ATOM_* */
  int32_t slot;
  int32_t slot2;    /* DIFF only */
  int32_t clause;   /* DNF clause 0..31 this atom belongs to */
  int32_t set_word; /* SET: first word in setwords[] */
  int32_t negate;   /* 1: atom result inverted */
  int64_t lo, hi;   /* RANGE/DIFF bounds, inclusive */
} scx_atom;

/* A predicate in disjunctive normal form over atoms[first .. first+n).
 * Row passes iff some clause c (bit c of clause_mask) has no failing atom.
 * clause_mask == 0 means TRUE. */
typedef struct scx_pred {
  int32_t first_atom;
  int32_t n_atoms;
  uint32_t clause_mask;
  int32_t _pad;
} scx_pred;

/* factor = a + b * v[slot]   (slot < 0: the constant a) */
typedef struct scx_factor {
  int64_t a, b;
  int32_t slot;
  int32_t _pad;
} scx_factor;

typedef struct scx_term {
  int64_t coef;
  int32_t n_factors;   /* 0..3 */
  int32_t _pad;
  scx_factor f[3];
} scx_term;

/* measure value per row = sum_t coef_t * prod_f factor_f, gated by cond_atom */
typedef struct scx_measure {
  int32_t op;          /* SCX_AGG_* (COUNT ignores terms) */
  int32_t n_terms;     /* 1..2 */
  int32_t cond_atom;   /* -1 or index into atoms[]: row contributes iff it holds */
  int32_t _pad;
  scx_term t[2];
} scx_measure;

/* key spec shared by probes, builds, group keys and partitioning:
 * packed = sum_k (f_k(v[slot_k]) - lo_k) << shift_k  (must fit 64 bits),
 * f_k = identity or the xform of component k (group keys only). */
typedef struct scx_keyspec {
  int32_t n;
  int32_t slot[SCX_MAX_KEYS];
  int32_t shift[SCX_MAX_KEYS];
  int32_t bits[SCX_MAX_KEYS];  /* component k must lie in [0, 2^bits_k)   */
  int32_t xform;               /* byte k: SCX_XFORM_* applied to v[slot_k] */
  int64_t lo[SCX_MAX_KEYS];
} scx_keyspec;

/* Lookup table built by scx_table_build and probed inside a pipeline. */
typedef struct scx_lookup {
  int32_t kind;        /* SCX_HT_HASH / SCX_HT_DIRECT */
  int32_t _pad;        /* BITMAP: coarse shift + 1 (0 = no coarse level)  */
  uint64_t keys;       /* HASH: u64[cap], SCX_EMPTY_KEY = free;
                          BITMAP: coarse bitmap (see scx_bitmap_coarsen),
                          staged in shared memory by the probing kernel */
  uint64_t vals;       /* u32[cap] build row, SCX_NO_ROW = free        */
  uint64_t cap;        /* HASH: power of two; DIRECT: key range size   */
} scx_lookup;

typedef struct scx_probe {
  int32_t kind;        /* SCX_JOIN_* */
  int32_t n_payload;
  scx_keyspec key;     /* probe-side key slots, same packing as the build */
  scx_lookup table;
  scx_column payload[SCX_MAX_PAYLOAD];   /* build-side columns, gathered ... */
  int32_t payload_slot[SCX_MAX_PAYLOAD]; /* ... into these operand slots     */
  scx_pred after;      /* filter applied right after this probe (atoms on
                          slots available at this stage)                  */
} scx_probe;

typedef struct scx_sink {
  int32_t kind;        /* SCX_SINK_* */
  int32_t n_measures;
  scx_measure m[SCX_MAX_MEASURES];
  /* group keys: DENSE uses card/lut (cell = mixed radix of ranks),
   *             HASH packs them with gkey (shift/lo). */
  scx_keyspec gkey;
  int32_t gcard[SCX_MAX_GKEYS];   /* DENSE: domain size of key k          */
  int32_t glut[SCX_MAX_GKEYS];    /* DENSE: offset into lut[] or -1       */
  int32_t n_cells;                /* DENSE: prod(gcard); HASH: 1 = direct-
                                     addressed (slot = packed key, gcap =
                                     key domain), 2 = direct with u32
                                     sum/count words, 0 = open addressing */
  int32_t n_out;                  /* COMPACT: output columns              */
  uint64_t acc;        /* DENSE: {u64 lo, i64 hi}[cells][M]; HASH: i64[cap][M] */
  uint64_t gkeys;      /* HASH: u64[cap] packed group keys                 */
  uint64_t gcap;       /* HASH: capacity (power of two)                    */
  uint64_t flags;      /* u32[4]: [0] hash table full, [1] dup build key   */
  int32_t out_slot[SCX_MAX_OUT];  /* COMPACT: slot, or -1 = base row index  */
  scx_column out[SCX_MAX_OUT];
  uint64_t status;     /* COMPACT: u64[n_tiles] look-back words, zeroed    */
  uint64_t count;      /* COMPACT/COUNT: u64[1] selected rows (written)    */
} scx_sink;

typedef struct scx_pipeline {
  int64_t n_rows;
  int32_t n_base;
  int32_t n_slots;
  int32_t n_probes;
  int32_t _pad;                  /* hint: estimated % of rows passing the first
                                    filtering stage (0 = unknown); tiling only */
  scx_column base[SCX_MAX_BASE];
  int32_t slot_dtype[SCX_MAX_SLOTS];
  scx_pred pre;                  /* on base slots, before probes          */
  scx_pred post;                 /* on any slot, after probes             */
  scx_probe probe[SCX_MAX_PROBES];
  scx_sink sink;
  scx_atom atoms[SCX_MAX_ATOMS];
  scx_measure polys[SCX_MAX_POLYS];  /* operands of SCX_ATOM_POLY atoms      */
  uint32_t setwords[SCX_MAX_SETWORDS];
  int16_t lut[SCX_MAX_LUT];
} scx_pipeline;

/* ---- library info ------------------------------------------------------ */
const char* scx_last_error(void);
int scx_abi_version(void);
/* kernels launched through libscx in this process so far */
uint64_t scx_launch_count(void);
/* sizeof of each descriptor struct, for binding checks: which = 0 pipeline,
 * 1 probe, 2 sink, 3 measure, 4 atom, 5 keyspec, 6 lookup */
int64_t scx_sizeof(int which);
/* number of SMs / opt-in smem on `device` (for host-side sizing) */
int scx_device_info(int device, int* sm_count, int* smem_optin);

/* ---- fused scan pipeline -------------------------------------------------
 * Replaces the numpy bodies of: ColumnTable.filter/take + driver predicate
 * expressions (table.py:171-192, queries.py:39-234), local_hash_join probe
 * (relops.py:59-94), group_aggregate (relops.py:97-160), q1's np.add.at grid
 * (queries.py:42-54) and q6's filtered sum (queries.py:105-119).
 * One launch: TMA-bulk-staged column tiles -> predicate -> probes ->
 * post-predicate -> sink.  `desc_host` is copied into the launch. */
int scx_pipeline_run(const scx_pipeline* desc_host, void* stream);
/* number of 'status' words a COMPACT sink needs for n_rows */
int64_t scx_pipeline_status_words(const scx_pipeline* desc_host);
/* The pipeline is specialised per descriptor: libscx generates CUDA C++ for
 * the plan (every dtype, literal, set, key packing and measure as an
 * immediate), compiles it with NVRTC for sm_100a and caches the cubin in
 * memory and on disk (<libdir>/jit_cache or $SCX_JIT_CACHE).  SCX_JIT=0
 * selects the descriptor-interpreting kernel instead (A/B baseline).
 * scx_pipeline_source: the generated source (length returned; up to cap-1
 * bytes + NUL copied to buf).  scx_pipeline_compile: codegen + NVRTC into
 * the disk cache without a device.  scx_jit_stats: kernels compiled / loaded
 * from disk / reused in memory by this process. */
int64_t scx_pipeline_source(const scx_pipeline* desc_host, char* buf, int64_t cap);
int scx_pipeline_compile(const scx_pipeline* desc_host);
int scx_jit_stats(int64_t* compiled, int64_t* disk_hits, int64_t* mem_hits);
/* Drop the memoised launch plans (tuning runs that change SCX_* codegen knobs
 * in-process; compiled kernels stay cached by source). */
int scx_jit_clear_plans(void);

/* ---- lookup tables (local_hash_join build side, relops.py:81-84) --------
 * Inserts packed keys of rows [0, n) of `cols` into `table` (pre-cleared
 * with scx_lookup_clear).  flags_dev[1] is set to 1 when a key repeats
 * (caller then uses the multi-match path). */
int scx_lookup_clear(const scx_lookup* table, void* stream);
int scx_lookup_build(const scx_lookup* table, const scx_column* cols, int n_cols,
                     const scx_keyspec* key, int64_t n, uint32_t* flags_dev,
                     void* stream);

/* ---- group table finalize (group_aggregate output, relops.py:115-160) ----
 * DENSE: folds n_ranks partial accumulator copies (stride cells*M*2 words)
 * per (cell, measure): ops_host[measure] 0 = exact 128-bit {lo,hi} sum,
 * 1 = min / 2 = max of the int64 in lo (collectives.py:198-206 semantics,
 * engine.py:342-343 all_reduce_sum).
 * HASH: compacts occupied slots -> out_keys (u64) + out_acc measure-major
 * (out_acc[m * cap + row]), count in count_dev[0].  Row order is slot order
 * (caller sorts by packed key). */
int scx_dense_reduce(const int64_t* acc_dev, int n_ranks, int cells, int m,
                     const int* ops_host, int64_t* out_dev, void* stream);
int scx_hash_agg_compact(const uint64_t* gkeys_dev, const int64_t* acc_dev,
                         int64_t cap, int m, uint64_t* out_keys_dev,
                         int64_t* out_acc_dev, uint64_t* count_dev, void* stream);

/* Ordered compaction of a direct-addressed group table (sink n_cells = 1):
 * occupied slots in slot order, i.e. already sorted by packed group key, so
 * no sort follows.  Same outputs as scx_hash_agg_compact; temp_dev sized by
 * scx_direct_agg_workspace(cap). */
int64_t scx_direct_agg_workspace(int64_t cap);
int scx_direct_agg_compact(const uint64_t* gkeys_dev, const int64_t* acc_dev, int64_t cap, int m,
                           uint64_t* out_keys_dev, int64_t* out_acc_dev, uint64_t* count_dev,
                           void* temp_dev, void* stream);

/* Same, for a direct table written without a key array (the JIT hash sink
 * with sink.gkeys == 0 in direct mode): slot e is a group iff its count word
 * acc[e*m + occ_word] > 0, and its packed key is e.  Replaces the same
 * np.unique/bincount step as scx_direct_agg_compact (relops.py:117-129). */
int scx_direct_agg_compact_counted(const int64_t* acc_dev, int64_t cap, int m, int occ_word,
                                   uint64_t* out_keys_dev, int64_t* out_acc_dev,
                                   uint64_t* count_dev, void* temp_dev, void* stream);

/* Same with a HAVING range on one measure word folded into the compaction:
 * slot e is kept iff its count word > 0 and hv_lo <= acc[e*m + hv_word] <=
 * hv_hi (Q18's sum(l_quantity) > 300: 150M groups scanned, ~600 written).
 * Equivalent to filtering the group_aggregate output (relops.py:97-160 then
 * table.py:174-177). */
/* One-pass, UNORDERED variant of scx_direct_agg_compact_having (warp-
 * aggregated atomics) for selective HAVING; the caller sorts the few
 * surviving packed keys.  Same outputs layout (out_acc[j*cap + g]). */
int scx_direct_agg_select_having(const int64_t* acc_dev, int64_t cap, int m, int occ_word,
                                 int hv_word, int64_t hv_lo, int64_t hv_hi,
                                 uint64_t* out_keys_dev, int64_t* out_acc_dev,
                                 uint64_t* count_dev, void* stream);
int scx_direct_agg_compact_having(const int64_t* acc_dev, int64_t cap, int m, int occ_word,
                                  int hv_word, int64_t hv_lo, int64_t hv_hi,
                                  uint64_t* out_keys_dev, int64_t* out_acc_dev,
                                  uint64_t* count_dev, void* temp_dev, void* stream);

/* Dense ranks of a non-decreasing key column (a clustered key: lineitem and
 * its materialised subsets by l_orderkey): rank_dev[i] = number of distinct
 * keys in key[0..i] - 1, keys_by_rank_dev[r] = (key of rank r) - lo,
 * count_dev[0] = number of distinct keys, count_dev[1] = number of positions
 * with key[i] < key[i-1] (non-zero: the column is not sorted and the ranks
 * are meaningless).  A group-by on such a key then uses a
 * direct table of exactly that many slots instead of hashing (replaces the
 * np.unique codes of relops.py:117-119 for sorted keys).  temp_dev sized by
 * scx_sorted_rank_workspace(n). */
int64_t scx_sorted_rank_workspace(int64_t n);
int scx_sorted_rank(const scx_column* key, int64_t n, int64_t lo, uint32_t* rank_dev,
                    uint64_t* keys_by_rank_dev, uint64_t* count_dev, void* temp_dev,
                    void* stream);

/* Coarse level of a membership bitmap: bit j of coarse_dev = OR of fine bits
 * [j << shift, (j+1) << shift) over nbits fine bits (rounded up to whole
 * words).  A probing kernel keeps it in shared memory and reads the fine
 * bitmap only when the coarse bit is set (the np.isin of relops.py:75 for
 * selective semi joins). */
int scx_bitmap_coarsen(const uint32_t* fine_dev, int64_t nbits, int shift, uint32_t* coarse_dev,
                       void* stream);

/* Top-k support (ColumnTable.sort_by(...).head(k), table.py:179-214):
 * scx_range_hist counts keys in [lo, hi) by the 8-bit digit ((key - lo) >>
 * shift) & 255 into counts_dev[256] (zeroed here); scx_select_below writes the
 * (key, row) pairs with key < T in row order (stable) and their number.  A
 * radix select narrows [lo, hi) until few rows lie below the k-th key, which
 * are then sorted instead of the whole input.  temp_dev sized by
 * scx_select_below_workspace(n). */
int scx_range_hist(const uint64_t* keys_dev, int64_t n, uint64_t lo, uint64_t hi, int shift,
                   uint32_t* counts_dev, void* stream);
int64_t scx_select_below_workspace(int64_t n);
int scx_select_below(const uint64_t* keys_dev, int64_t n, uint64_t T, uint64_t* out_keys_dev,
                     uint32_t* out_idx_dev, uint64_t* count_dev, void* temp_dev, void* stream);

/* Stream aggregation over a non-decreasing key column (relops.py:97-160 for
 * clustered input, e.g. lineitem by l_orderkey): each group is aggregated by
 * the thread holding its first row; no group table.  vals/ops: m plain
 * columns with SCX_AGG_* (COUNT ignores its column); optional HAVING
 * hv_lo <= acc[hv] <= hv_hi (hv = -1: none).  Writes *count groups (unordered)
 * as out_keys[g] (raw key values) and out_acc[j*cap + g]; *overflow = 1 if
 * more than cap groups qualified.  scx_is_sorted: *bad = #{i: key[i] < key[i-1]}. */
int scx_is_sorted(const scx_column* col, int64_t n, uint64_t* bad_dev, void* stream);
int scx_sorted_group_agg(const scx_column* key, const scx_column* vals, const int* ops, int m,
                         int64_t n, int hv, int64_t hv_lo, int64_t hv_hi, int64_t* out_keys_dev,
                         int64_t* out_acc_dev, int64_t cap, uint64_t* count_dev,
                         uint32_t* overflow_dev, void* stream);

/* Narrow direct group tables (sink.n_cells == 2: u32 count / small-sum
 * accumulators, half the random-access footprint of int64) are widened to
 * int64 words before scx_direct_agg_compact_counted. */
int scx_widen_u32(const uint32_t* in_dev, int64_t n, int64_t* out_dev, void* stream);

/* 128-bit {lo, hi} hash-group sums (measure._pad = 1 marks a "wide" sum whose
 * accumulator is two words) -> int64; flag_dev[0] |= 1 if any value does not
 * fit (group_aggregate output, relops.py:138-158). */
int scx_i128_narrow(const int64_t* lo_dev, const int64_t* hi_dev, int64_t n, int64_t* out_dev,
                    uint32_t* flag_dev, void* stream);

/* ---- key unpack / convert ------------------------------------------------ */
/* out[i] = ((packed[i] >> shift) & mask) + lo, stored as dtype */
int scx_unpack_key(const uint64_t* packed_dev, int64_t n, int shift, uint64_t mask,
                   int64_t lo, scx_column out, void* stream);
/* out_f64[i] = (double)in[i*stride] / 10^scale  (optionally / max(cnt,1)) */
int scx_fixed_to_f64(const int64_t* in_dev, int64_t stride, int64_t n, int scale,
                     const int64_t* count_dev, int64_t count_stride,
                     double* out_dev, void* stream);

/* ---- sort (ColumnTable.sort_by, table.py:198-214) -------------------------
 * Stable LSD radix sort of (key u64, value u32) pairs on key bits
 * [0, n_bits).  Ping-pong buffers; result lands in *_out.  temp_dev sized by
 * scx_sort_workspace. */
int64_t scx_sort_workspace(int64_t n);
int scx_sort_pairs(const uint64_t* keys_in, const uint32_t* vals_in,
                   uint64_t* keys_out, uint32_t* vals_out,
                   uint64_t* keys_tmp, uint32_t* vals_tmp,
                   int64_t n, int n_bits, void* temp_dev, void* stream);
/* key[i] = encode(col[idx ? idx[i] : i]) : order-preserving u64 of the value,
 * minus lo, bit-inverted within n_bits when descending. */
int scx_encode_sort_key(scx_column col, const uint32_t* idx_dev, int64_t n,
                        int64_t lo, int n_bits, int descending, int shift,
                        const int32_t* lut_dev, uint64_t* key_dev, int accumulate,
                        void* stream);
/* out_dev[0] = min, out_dev[1] = max over the column (integer dtypes);
 * out_dev must be pre-set to {INT64_MAX, INT64_MIN}. */
int scx_minmax(scx_column col, int64_t n, int64_t* out_dev, void* stream);
/* out[i] = in[idx[i]] for a column of dtype (take, table.py:76-77/171) */
int scx_gather(scx_column in, const uint32_t* idx_dev, int64_t n, scx_column out,
               void* stream);
/* idx[i] = i */
int scx_iota(uint32_t* idx_dev, int64_t n, void* stream);
/* p[i * stride] = value for i < n  (table / accumulator initialisation) */
int scx_fill_i64(int64_t* p_dev, int64_t n, int64_t stride, int64_t value, void* stream);
/* p[r * w + j] = pattern_host[j] for r < rows, j < w <= 16: a row-major
 * group table's identities in one pass */
int scx_fill_rows(int64_t* p_dev, int64_t rows, int w, const int64_t* pattern_host, void* stream);
/* dst_host[0..nbytes) = src_dev[0..nbytes) by a kernel storing into mapped
 * pinned host memory (cudaHostAlloc'ed: UVA-mapped): a small result read that
 * does not queue on a copy engine behind an in-flight upload.  No reference
 * counterpart (the reference's results are host numpy arrays already). */
int scx_write_mapped(const void* src_dev, void* dst_host, int64_t nbytes, void* stream);

/* ---- hash partitioning (exchange.py:35-70) --------------------------------
 * bucket(row) = fib_hash(keys) mod n_parts with the reference's u64 wrap:
 *   acc = 0; for k: acc = (acc ^ (u64(v_k) * F)) * F,  F = 0x9E3779B97F4A7C15
 * scx_hash_keys writes the raw u64 hashes.  scx_partition computes counts
 * (u64[n_parts]) and a stable scatter of every column into `outs`, parts
 * contiguous in bucket order, rows in input order within a part. */
int scx_hash_keys(const scx_column* keys, int n_keys, int64_t n, uint64_t* out_dev,
                  void* stream);
int64_t scx_partition_workspace(int64_t n, int n_parts);
int scx_partition(const scx_column* keys, int n_keys, const scx_column* cols,
                  const scx_column* outs, int n_cols, int64_t n, int n_parts,
                  uint64_t* counts_dev, void* temp_dev, void* stream);

/* ---- shuffle partition to arbitrary destinations (exchange.py:131-174) ----
 * Pass 1 (scx_part_hist): bucket = fib_hash(keys) mod n_parts; per-part row
 * totals to counts_dev (u64[n_parts]) and per-(part, CTA) stable offsets kept
 * in ws (sized by scx_part_workspace; n_parts <= 64).
 * Pass 2 (scx_part_scatter, same ws): every column's rows of part d are
 * written, in source row order, to dst_dev[c * n_parts + d] (a device array
 * of byte addresses: the receiver-side slot of this source in worker d's
 * buffer -- local memory, a peer GPU's HBM, or another virtual rank's buffer
 * on the same device).  scx_partition is pass 1 + pass 2 into a contiguous
 * local layout. */
int64_t scx_part_workspace(int64_t n, int n_parts);
int scx_part_hist(const scx_column* keys, int n_keys, int64_t n, int n_parts, void* ws_dev,
                  uint64_t* counts_dev, void* stream);
int scx_part_scatter(const scx_column* keys, int n_keys, const scx_column* cols, int n_cols,
                     int64_t n, int n_parts, const uint64_t* dst_dev, const void* ws_dev,
                     void* stream);

/* ---- multi-match inner join (relops.py:59-94: stable argsort +
 * searchsorted + repeat) ----------------------------------------------------
 * lkeys: packed u64 join key per LEFT row; rsorted: the RIGHT side's packed
 * keys sorted stably (scx_sort_pairs, values = right row ids = rperm).
 * scx_join_match fills the workspace (per-left-row match run + exclusive
 * scan) and writes the pair count to total_dev (u64, device).
 * scx_join_expand writes the pairs in left row order, matches in right row
 * order (out_l / out_r: u32[total]).  ws sized by scx_join_workspace(n). */
int64_t scx_join_workspace(int64_t n);
int scx_join_match(const uint64_t* lkeys_dev, int64_t n, const uint64_t* rsorted_dev, int64_t m,
                   void* ws_dev, uint64_t* total_dev, void* stream);
int scx_join_expand(const void* ws_dev, int64_t n, const uint32_t* rperm_dev, int64_t total,
                    uint32_t* out_l_dev, uint32_t* out_r_dev, void* stream);

/* ---- dictionary reconciliation (exchange.py:177-192, 217-251) -------------
 * out[i] = lut[in[i]] (dictionary codes through a rank's remap into the
 * union dictionary); a code outside [0, lut_n) sets *bad_dev = 1. */
int scx_remap_codes(scx_column in, int64_t n, const int32_t* lut_dev, int32_t lut_n,
                    scx_column out, int* bad_dev, void* stream);

/* ---- NCCL data plane of the exchanges (process-per-GPU jobs) ---------------
 * Communicators are opaque handles (ncclComm_t).  Counts / offsets / sizes
 * are HOST arrays of length nranks; all transfers are asynchronous on
 * `stream`.  Replaces: exchange.py:73-97 size_exchange and 131-174
 * shuffle_table (scx_alltoallv: one group of ncclSend/ncclRecv, the paper's
 * Alg. 1), exchange.py:195-285 broadcast_table (scx_bcast_group: the N root
 * broadcasts of a column in ONE group, Alg. 2), collectives.py:199-213
 * all_reduce on exact integers (scx_allreduce_i64, op 0 sum / 1 min / 2 max),
 * engine.py:345-365 gather (scx_gather_to0). */
int scx_nccl_version(int* version);
int64_t scx_comm_id_bytes(void);
int scx_comm_unique_id(void* id_out);
int scx_comm_init_rank(void** comm_out, int nranks, const void* id, int rank);
int scx_comm_init_all(int n, const int* devs, void** comms_out);
int scx_comm_destroy(void* comm);
int scx_alltoallv(void* comm, const void* send_dev, const int64_t* send_counts,
                  const int64_t* send_offs, void* recv_dev, const int64_t* recv_counts,
                  const int64_t* recv_offs, int elem_bytes, void* stream);
int scx_bcast_group(void* comm, void* const* bufs_dev, const int64_t* bytes, int n_roots,
                    void* stream);
int scx_allreduce_i64(void* comm, const int64_t* send_dev, int64_t* recv_dev, int64_t count,
                      int op, void* stream);
int scx_gather_to0(void* comm, const void* send_dev, int64_t bytes, void* const* recv_dev,
                   const int64_t* recv_bytes, void* stream);

/* ---- packed host columns: the load path's H2D bytes (data.py:284-302
 * partition_dataset / the cold run) ---------------------------
 * The reference hands float64/int64 columns to its workers; here a host
 * column is sent bit-packed and unpacked on the device into its narrowed
 * layout.  SCX_PACK_FOR: value = lo + field (k bits); SCX_PACK_DELTA
 * (non-decreasing columns): blocks of scx_pack_delta_block() rows, value =
 * bases[block] + running sum of the block's fields (first field 0);
 * SCX_PACK_IOTA (surrogate keys): value = lo + row, no words.  Field i sits at
 * bits [i*k, i*k+k) of a little-endian u32 word stream of scx_pack_words(n, k)
 * words (one padding word).  scx_pack_host is host code (threads), k <= 32. */
#define SCX_PACK_FOR   0
#define SCX_PACK_DELTA 1
#define SCX_PACK_IOTA  2
int64_t scx_pack_words(int64_t n, int k);
int64_t scx_pack_delta_block(void);
int scx_pack_host(const void* in, int dtype, int64_t n, int64_t lo, int k, int delta,
                  uint32_t* out_words, int64_t* out_bases, int n_threads);
int scx_unpack(const uint32_t* words_dev, int64_t n, int k, int64_t lo, int encoding,
               const int64_t* bases_dev, scx_column out, void* stream);
/* Column-relative packing (the host packs value - ref[i] - lo in k bits):
 * out[i] = ref[i] + lo + field; ref is an already unpacked column of the same
 * table (l_receiptdate against l_shipdate: 5 bits instead of 12). */
int scx_unpack_diff(const uint32_t* words_dev, int64_t n, int k, int64_t lo, scx_column ref,
                    scx_column out, void* stream);
/* key-relative unpack: out[i] = ref[fk[i] - fk_lo] + lo + field(words, i, k),
 * ref a dense-keyed parent column of ref_n rows (a child date stored against
 * its parent row's date through the foreign key fk).  Extension of the load
 * path (codec.py); no reference counterpart. */
int scx_unpack_fkdiff(const uint32_t* words, int64_t n, int k, int64_t lo, scx_column fk,
                      int64_t fk_lo, scx_column ref, int64_t ref_n, scx_column out, void* stream);
/* key-indexed unpack: out[i] = ref[(fk[i] - fk_lo) * fanout + field(words, i, k)],
 * ref a parent column grouped by a dense key with `fanout` rows per key (a
 * child value that is one of its parent group's values: l_suppkey among the
 * partsupp suppliers of l_partkey).  Load-path extension; no reference
 * counterpart. */
int scx_unpack_fkidx(const uint32_t* words, int64_t n, int k, scx_column fk, int64_t fk_lo,
                     int64_t fanout, scx_column ref, int64_t ref_n, scx_column out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SCX_H */
