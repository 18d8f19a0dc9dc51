/*
 * prefixopt_cuda.h — C ABI of the B200 (sm_100a) GGR reorder + PHC path.
 *
 * This is the drop-in boundary for the reference's hot path
 * (`prefixopt::ggr`, `phc`, `hit`, `sort_rows_fixed_order`, `compute_stats`,
 * `fixed_order_by_hitcount_stats`, `fixed_order_by_stats`). The reference has
 * no FFI of its own (it is a header-only C++20 library); the
 * entry points below are what a binding for that API needs: plain pointers
 * and sizes, no C++ or torch types. The C++ headers under proj/include/
 * prefixopt/ and the Python package paper_2403_05821_b200 both sit on top
 * of these functions.
 *
 * Conventions
 *   - A table is a row-major grid of byte strings: cell (r, f) is
 *     arena[offsets[r*m+f] .. offsets[r*m+f+1]). Arena/offsets live on the
 *     host or on the current CUDA device (po_table.location). Host inputs are
 *     copied to the device inside the call.
 *   - Every function returns PO_OK or an error code; po_last_error() returns
 *     the message for the calling thread. Error codes mirror the reference's
 *     exception taxonomy (errors.hpp:10-42) so a wrapper can rethrow the same
 *     class.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream). Calls are
 *     synchronous with respect to the host: outputs are valid on return.
 *   - Calls are re-entrant across host threads; each call owns its scratch.
 */
#ifndef PREFIXOPT_CUDA_H
#define PREFIXOPT_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:10-42) ----------------------------------- */
#define PO_OK 0
#define PO_ERR_ERROR 1        /* prefixopt::error (also CUDA failures)      */
#define PO_ERR_SCHEMA 2       /* prefixopt::schema_error                    */
#define PO_ERR_STRUCTURAL 3   /* prefixopt::structural_error                */
#define PO_ERR_DOMAIN 4       /* prefixopt::domain_error                    */
#define PO_ERR_SIZE 5         /* prefixopt::size_error                      */
#define PO_ERR_IO 6           /* prefixopt::io_error                        */
#define PO_ERR_OUT_OF_RANGE 7 /* std::out_of_range (Table::cell .at())      */
#define PO_ERR_INVALID_ARG 8  /* bad ABI usage (null pointers, bad enum)    */

/* ---- enums (tokenizer.hpp:40-96, scoring.hpp:20, ggr.hpp:25-29) -------- */
#define PO_LOC_HOST 0
#define PO_LOC_DEVICE 1

#define PO_TOK_CHAR 0   /* CharTokenizer::count  (tokenizer.hpp:44)        */
#define PO_TOK_WORD 1   /* WordTokenizer::count  (tokenizer.hpp:64-73)     */
#define PO_TOK_CUSTOM 2 /* lengths supplied in po_table.cell_lens          */

#define PO_SCORE_VALUE 0    /* SegmentScoring::value_only                  */
#define PO_SCORE_FRAGMENT 1 /* SegmentScoring::full_fragment               */

#define PO_STATS_WEIGHTED 0 /* cardinality_weighted_squared (default)      */
#define PO_STATS_SQUARED 1  /* squared_length                              */
#define PO_STATS_LENFREQ 2  /* length_frequency                            */

/* Table view. Replaces prefixopt::Table (table.hpp:24-104) at the boundary. */
typedef struct po_table {
  uint64_t n_rows;
  uint32_t n_fields;
  uint32_t location;               /* PO_LOC_* of arena / offsets / cell_lens */
  const char* const* field_names;  /* host, n_fields entries                  */
  const uint64_t* field_name_lens; /* host, byte length of each name          */
  const uint8_t* arena;            /* cell bytes                               */
  const uint64_t* offsets;         /* n_rows*n_fields + 1, row-major           */
  const uint64_t* cell_lens;       /* PO_TOK_CUSTOM only: per-cell segment
                                      length (tok.count of the value, or of the
                                      fragment in full_fragment mode), else NULL */
} po_table;

/* GgrConfig (ggr.hpp:48-54). */
typedef struct po_ggr_config {
  uint64_t row_recursion_depth;     /* default 4      */
  uint64_t column_recursion_depth;  /* default 2      */
  uint64_t hitcount_stop_threshold; /* default 100000 */
  int32_t use_fds;                  /* default 1      */
  int32_t stats_variant;            /* PO_STATS_*     */
} po_ggr_config;

/* FunctionalDependencySet (fd.hpp:21-26) with names already resolved to
 * field indices by the caller (Table::require_field, ggr.hpp:158). */
typedef struct po_fd_groups {
  uint32_t n_groups;
  const uint32_t* group_offsets; /* n_groups + 1 */
  const int32_t* members;        /* field indices */
} po_fd_groups;

/* SolveStats (solve_result.hpp:9-14). */
typedef struct po_solve_stats {
  uint64_t recursive_calls;
  uint64_t candidates_examined;
  uint64_t max_depth;
  double wall_ms;
} po_solve_stats;

/* ---- entry points ------------------------------------------------------ */

/* prefixopt::ggr (ggr.hpp:367-394). Emits the schedule (row ids in request
 * order, and a full field permutation per request: n_rows*n_fields ints),
 * its PHC and the solver counters. Outputs live at `out_location`. FD
 * groups sharing two members: PO_ERR_SIZE, see po_ggr_schedule. */
int po_ggr(const po_table* t, const po_fd_groups* fds, const po_ggr_config* cfg,
           int32_t tokenizer, int32_t scoring, uint32_t out_location,
           uint64_t* out_row_ids, int32_t* out_field_orders, uint64_t* out_phc,
           po_solve_stats* out_stats, void* stream);

/* prefixopt::ggr returning the schedule as a handle with CSR field orders.
 * Needed when FD groups share members: the reference then emits a partner
 * once per group holding it, so field orders can be longer than n_fields
 * (ggr.hpp:154-164, 280-282; po_ggr fails with PO_ERR_SIZE in that case).
 * Same results as po_ggr otherwise. Device memory is owned by the handle. */
typedef struct po_schedule po_schedule;
int po_ggr_schedule(const po_table* t, const po_fd_groups* fds, const po_ggr_config* cfg,
                    int32_t tokenizer, int32_t scoring, po_schedule** out_schedule,
                    uint64_t* out_phc, po_solve_stats* out_stats, void* stream);
int po_schedule_info(const po_schedule* schedule, uint64_t* out_entries,
                     uint64_t* out_fields_total);
/* row ids (entries), CSR offsets (entries + 1) and fields (fields_total). */
int po_schedule_copy(const po_schedule* schedule, uint32_t out_location, uint64_t* out_row_ids,
                     uint64_t* out_order_offsets, int32_t* out_order_fields, void* stream);
void po_schedule_free(po_schedule* schedule);

/* prefixopt::phc (objective.hpp:94-99) over an arbitrary schedule: entry i is
 * row row_ids[i] rendered with fields order_fields[order_offsets[i] ..
 * order_offsets[i+1]). Schedule arrays live at `sched_location`. */
int po_phc(const po_table* t, int32_t tokenizer, int32_t scoring, uint64_t n_entries,
           const uint64_t* row_ids, const uint64_t* order_offsets,
           const int32_t* order_fields, uint32_t sched_location, uint64_t* out_phc,
           void* stream);

/* prefixopt::hit (objective.hpp:70-91): score of request r against r-1.
 * r >= n_entries -> PO_ERR_DOMAIN. */
int po_hit(const po_table* t, int32_t tokenizer, int32_t scoring, uint64_t n_entries,
           const uint64_t* row_ids, const uint64_t* order_offsets,
           const int32_t* order_fields, uint32_t sched_location, uint64_t r,
           uint64_t* out_hit, void* stream);

/* prefixopt::sort_rows_fixed_order (objective.hpp:154-171). `field_order`
 * (host) must be a permutation of the schema, else PO_ERR_SCHEMA. Writes the
 * n_rows row ids in request order at out_location. */
int po_sort_rows_fixed_order(const po_table* t, const int32_t* field_order,
                             uint32_t out_location, uint64_t* out_row_ids, void* stream);

/* prefixopt::compute_stats (stats.hpp:25-45): per field the exact number of
 * distinct raw values and the sum of segment lengths (host outputs). The
 * caller forms avg_len = double(total_len) / n_rows. */
int po_compute_stats(const po_table* t, int32_t tokenizer, int32_t scoring,
                     uint64_t* out_cardinality, uint64_t* out_total_len, void* stream);

/* prefixopt::fixed_order_by_hitcount_stats (ggr.hpp:59-84) and
 * fixed_order_by_stats (objective.hpp:176-188): host-only IEEE-double
 * ranking of fields from (total_rows, cardinality[], avg_len[]). */
int po_fixed_order_by_hitcount_stats(uint32_t n_fields, uint64_t total_rows,
                                     const uint64_t* cardinality, const double* avg_len,
                                     int32_t variant, int32_t* out_order);
int po_fixed_order_by_stats(uint32_t n_fields, uint64_t total_rows,
                            const uint64_t* cardinality, const double* avg_len,
                            int32_t* out_order);

/* Partition-signature comparison of field pairs: the core of
 * prefixopt::validate_fds (fd.hpp:66-109) and discover_fds (fd.hpp:114-141).
 * sig_f[r] = first row holding row r's value in field f (partition_signature,
 * fd.hpp:56-64). For pair k: out_first_diff[k] = first row r with
 * sig_{pair_a[k]}[r] != sig_{pair_b[k]}[r] (n_rows when the partitions are
 * identical); out_sig_a[k] / out_sig_b[k] = the two signatures at that row
 * (the witness rows). Host outputs; values compared as raw bytes. */
int po_fd_compare(const po_table* t, uint32_t n_pairs, const int32_t* pair_a,
                  const int32_t* pair_b, uint64_t* out_first_diff, uint64_t* out_sig_a,
                  uint64_t* out_sig_b, void* stream);

/* prefixopt::render_prompt (objective.hpp:102-131) of every entry of a
 * schedule (CSR field orders as in po_phc; arrays at sched_location):
 * prompt i = out_bytes[out_offsets[i] .. out_offsets[i+1]). Call with
 * out_bytes == NULL to get the total size in *out_total (out_offsets is
 * filled either way, n_entries + 1 values); then again with a buffer of at
 * least that many bytes (else PO_ERR_SIZE, checked before any byte is
 * written). Outputs at out_location; a device out_bytes is written in place
 * (any alignment; bytes past out_total are untouched), a size query only
 * computes lengths. A row or field outside the table -> PO_ERR_OUT_OF_RANGE
 * (Table::cell). */
int po_render_prompts(const po_table* t, uint64_t n_entries, const uint64_t* row_ids,
                      const uint64_t* order_offsets, const int32_t* order_fields,
                      uint32_t sched_location, const uint8_t* system_prompt,
                      uint64_t system_prompt_len, const uint8_t* question, uint64_t question_len,
                      uint32_t out_location, uint64_t* out_offsets, uint8_t* out_bytes,
                      uint64_t out_capacity, uint64_t* out_total, void* stream);

/* prefixopt::dedup (cost.hpp:171-186), byte-exact: strings
 * arena[offsets[i] .. offsets[i+1]) (i < n, at `location`). Host outputs:
 * out_expansion[i] = index of string i's unique; out_unique_first[u] =
 * original index of unique u (uniques in first-occurrence order, n slots);
 * *out_n_unique. */
int po_dedup(uint64_t n, const uint8_t* arena, const uint64_t* offsets, uint32_t location,
             uint64_t* out_expansion, uint64_t* out_unique_first, uint64_t* out_n_unique,
             void* stream);

/* prefixopt::simulate (cache_sim.hpp:223-285) with EvictionPolicy::none
 * (unbounded cache) over prompts arena[offsets[i] .. offsets[i+1]) (at
 * `location`) and the char or word tokenizer. Host outputs per request (n
 * slots each, any may be NULL): input tokens, credited hit (raw hit if >=
 * min_cacheable_prefix_tokens, else 0), miss = input - hit, written =
 * input - raw hit; out_totals[3] = total input, hit, miss. n == 0 ->
 * PO_ERR_DOMAIN (the reference's "prompt list is empty"). LRU eviction is
 * sequential by definition and has no GPU entry point. */
int po_replay_unbounded(uint64_t n, const uint8_t* arena, const uint64_t* offsets,
                        uint32_t location, int32_t tokenizer,
                        uint64_t min_cacheable_prefix_tokens, uint64_t* out_input_tokens,
                        uint64_t* out_hit_tokens, uint64_t* out_miss_tokens,
                        uint64_t* out_written_tokens, uint64_t* out_totals, void* stream);

/* prefixopt::load_csv (table.hpp:114-215): RFC-4180 text (at `location`)
 * parsed on the GPU into a table; same errors as the reference
 * (PO_ERR_STRUCTURAL: missing header row, unterminated quoted field, a line
 * with the wrong number of cells; PO_ERR_SCHEMA: duplicate header field,
 * empty field name). The handle owns the parsed table until po_csv_free. */
typedef struct po_csv po_csv;
int po_load_csv(const uint8_t* data, uint64_t len, uint32_t location, po_csv** out, void* stream);
int po_csv_info(const po_csv* csv, uint64_t* out_rows, uint32_t* out_fields,
                uint64_t* out_arena_bytes, uint64_t* out_names_bytes);
/* arena (arena_bytes), offsets (rows*fields + 1, row-major) at out_location;
 * names (names_bytes) and name_offsets (fields + 1) on the host. */
int po_csv_copy(const po_csv* csv, uint32_t out_location, uint8_t* out_arena,
                uint64_t* out_offsets, uint8_t* out_names, uint64_t* out_name_offsets,
                void* stream);
void po_csv_free(po_csv* csv);

/* prefixopt::load_jsonl (table.hpp:225-269): one JSON object per line (host
 * text), parsed on the host with the reference's JSON library (nlohmann 3.11.3):
 * union schema in first-seen key order, absent keys "", strings verbatim,
 * null "", other values their compact JSON text; blank lines skipped.
 * PO_ERR_STRUCTURAL: a line that does not parse ("jsonl: line N: ...") or is
 * not an object; PO_ERR_SCHEMA: an empty key. Handle as po_csv, host outputs. */
typedef struct po_jsonl po_jsonl;
int po_load_jsonl(const uint8_t* data, uint64_t len, po_jsonl** out);
int po_jsonl_info(const po_jsonl* j, uint64_t* out_rows, uint32_t* out_fields,
                  uint64_t* out_arena_bytes, uint64_t* out_names_bytes);
int po_jsonl_copy(const po_jsonl* j, uint8_t* out_arena, uint64_t* out_offsets, uint8_t* out_names,
                  uint64_t* out_name_offsets);
void po_jsonl_free(po_jsonl* j);

/* prefixopt::load_fd_config (fd.hpp:143-164): the FD config document
 * {"groups": [["field", ...], ...]} (host text). First call with the three
 * array pointers NULL for the sizes; then group g = names
 * [group_offsets[g], group_offsets[g+1]), name k = bytes
 * [name_offsets[k], name_offsets[k+1]). PO_ERR_STRUCTURAL: not JSON
 * ("fd config: ..."); PO_ERR_SCHEMA: wrong shape (the reference's messages). */
int po_load_fd_config(const uint8_t* data, uint64_t len, uint32_t* out_groups, uint64_t* out_names,
                      uint64_t* out_names_bytes, uint64_t* out_group_offsets,
                      uint64_t* out_name_offsets, uint8_t* out_bytes);

/* ---- row-sharded solve over several GPUs ---------------
 * No reference counterpart: the reference ggr() (ggr.hpp:367-394) is one
 * process on one table. Here every rank (one per GPU) passes a contiguous
 * range of the table's rows (rank 0 the first rows, rank 1 the next, ...);
 * the result is bit-identical to po_ggr on the whole table, delivered as one
 * contiguous slice of the schedule per rank (concatenating the slices in
 * rank order gives po_ggr's schedule; row ids are global). All ranks call
 * every po_ggr_sharded together (it is collective). */
typedef struct po_comm po_comm;   /* a rank's communicator                */
typedef struct po_slice po_slice; /* a rank's slice of a sharded schedule */

/* NCCL transport, one process per GPU: rank 0 creates the 128-byte id and
 * ships it to the other ranks (any side channel, e.g. torch.distributed). */
int po_comm_unique_id(uint8_t* out_id128);
int po_comm_init_nccl(const uint8_t* id128, int32_t nranks, int32_t rank, po_comm** out);
/* In-process transport: nranks communicators for nranks host threads of one
 * process (any devices, several ranks may share one GPU). */
int po_comm_init_local(int32_t nranks, po_comm** out_array);
/* Host-staged transport over caller-provided collectives on HOST buffers
 * (e.g. MPI, or torch.distributed with the gloo backend): every device
 * collective is staged D2H, handed to the callbacks, and staged back H2D.
 * Callbacks return 0 on success. Ranks are processes (or threads) of any
 * layout, including several ranks on one GPU. */
typedef struct po_host_collectives {
  void* ctx;
  /* recv = every rank's `bytes` bytes, back to back in rank order */
  int (*allgather)(void* ctx, const void* send, void* recv, uint64_t bytes);
  /* rank r contributes recv_bytes[r] bytes (send holds recv_bytes[rank]);
   * recv gets them back to back in rank order */
  int (*allgatherv)(void* ctx, const void* send, void* recv, const uint64_t* recv_bytes);
  /* send_bytes[r] bytes to rank r and recv_bytes[r] from rank r, both
   * contiguous in rank order */
  int (*alltoallv)(void* ctx, const void* send, const uint64_t* send_bytes, void* recv,
                   const uint64_t* recv_bytes);
} po_host_collectives;
int po_comm_init_host(const po_host_collectives* ops, int32_t nranks, int32_t rank, po_comm** out);
int po_comm_destroy(po_comm* comm);

/* Sharded prefixopt::ggr. `t` holds this rank's rows (same fields on every
 * rank). The slice handle owns device memory until po_slice_free. */
int po_ggr_sharded(po_comm* comm, const po_table* t, const po_fd_groups* fds,
                   const po_ggr_config* cfg, int32_t tokenizer, int32_t scoring,
                   po_slice** out_slice, uint64_t* out_phc, po_solve_stats* out_stats,
                   void* stream);
/* Position of the slice in the schedule and its number of requests. */
int po_slice_info(const po_slice* slice, uint64_t* out_offset, uint64_t* out_count);
/* Copies the slice: count global row ids and count*n_fields field indices. */
int po_slice_copy(const po_slice* slice, uint32_t out_location, uint64_t* out_row_ids,
                  int32_t* out_field_orders, void* stream);
void po_slice_free(po_slice* slice);

/* Test hook (not a reference function): the stable radix sort of the K8
 * row-key sorts, (u64 key, u32 value) pairs by key bits [begin, end), host
 * arrays in and out. */
int po_debug_radix_sort(const uint64_t* keys, const uint32_t* vals, uint64_t n, int32_t begin_bit,
                        int32_t end_bit, uint64_t* out_keys, uint32_t* out_vals);

/* Test hook (not a reference function): the stable merge sort of the K3
 * small-job sorts on (a, b, value) records, ordered by (a, b); host arrays. */
int po_debug_merge_sort(const uint64_t* a, const uint64_t* b, const uint32_t* vals, uint64_t n,
                        uint64_t* out_a, uint64_t* out_b, uint32_t* out_vals);

/* Thread-local message of the last failing call on this thread. */
const char* po_last_error(void);

/* Library/device info: compiled arch string, e.g. "sm_100a". */
const char* po_build_info(void);

/* Number of CUDA kernels this library launched in this process (counter
 * incremented at each launch site; used by bench.py's gpu_launches). */
uint64_t po_kernel_launch_count(void);

/* Large transient device buffers are kept in a per-device block cache
 * between calls (no memory is mapped on repeated calls). po_trim_device_cache
 * returns the idle blocks of every device to the driver; the returned value
 * is the number of bytes released. Safe to call at any time; blocks in use by
 * a running call are kept. */
uint64_t po_trim_device_cache(void);

/* Per-kernel CUDA-event timing on the launching stream. po_profile_report
 * drains the recorded launches and writes "name count total_ms" lines into
 * buf (NUL-terminated, truncated to cap); returns the full length + 1. */
void po_profile_enable(int enable);
uint64_t po_profile_report(char* buf, uint64_t cap);

#ifdef __cplusplus
}
#endif

#endif /* PREFIXOPT_CUDA_H */
