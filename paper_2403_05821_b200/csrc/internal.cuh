// Internal interfaces between the translation units of libprefixopt_cuda.so.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "common.cuh"

namespace po {

class Comm;

// Escaped fragment-key order of bytes (refine.cu): code[b] = rank of byte b's
// json_escape expansion, code[256] = rank of the closing '"'.
void esc_code_table(uint16_t code[257]);

// Device view of the caller's table (arena/offsets already in HBM).
struct DeviceTable {
  uint64_t n = 0;
  uint32_t m = 0;
  std::vector<std::string> names;  // host
  const uint8_t* arena = nullptr;  // device
  uint64_t arena_bytes = 0;
  const uint64_t* offsets = nullptr;  // device, n*m+1
  const uint64_t* cell_lens = nullptr;  // device or null (custom tokenizer)
  // deferred host table (make_device_table(stream_host = true)): arena and
  // offsets stay in host memory and the dictionary pass streams row chunks
  // (arena / offsets above are then null)
  const uint8_t* h_arena = nullptr;
  const uint64_t* h_offsets = nullptr;
  // owned copies when the caller passed host buffers
  DevBuf<uint8_t> own_arena;
  DevBuf<uint64_t> own_offsets;
  DevBuf<uint64_t> own_lens;
};

// Builds a DeviceTable from the ABI view, copying host buffers to HBM (or,
// with stream_host, leaving arena + offsets on the host for the streamed
// dictionary pass: only for callers that use the table through encode()).
void make_device_table(const po_table* t, int tok, cudaStream_t s, DeviceTable& out,
                       bool stream_host = false);

// A second stream of the calling thread (current device) for copies that
// overlap work on the call's stream.
cudaStream_t copy_stream();
cudaStream_t aux_stream();  // per-thread, per-device side stream for overlapped work

void exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, cudaStream_t s);

// Stable LSD radix sort of (u64 key, u32 value) pairs by key bits
// [begin_bit, end_bit) (radix.cu: hand-written onesweep). kin/vin and
// kout/vout must not overlap. PO_RADIX=cub routes to cub::DeviceRadixSort
// (comparison runs).
void debug_merge_sort(const uint64_t* a, const uint64_t* b, const uint32_t* v, uint32_t n,
                      uint64_t* oa, uint64_t* ob, uint32_t* ov, cudaStream_t s);
void radix_sort_pairs(const uint64_t* kin, uint64_t* kout, const uint32_t* vin, uint32_t* vout,
                      uint32_t n, int begin_bit, int end_bit, cudaStream_t s);

// K1 + K2 (dict.cu): exact per-column dictionaries in one read of the cell
// bytes. cid_mat[r*m + c] = dense id of cell (r, c)'s value within column c
// in first-claim order; distinct value d = colbase[c] + id is the string
// val_arena[val_off[d] .. + val_len[d]) held by row rep_row[d].
struct DictResult {
  uint64_t D = 0;
  std::vector<uint64_t> card, colbase;
  DevBuf<uint64_t> d_colbase;
  DevBuf<uint64_t> val_off;
  DevBuf<uint32_t> val_len, rep_row, d_col;
  const uint8_t* val_arena = nullptr;  // the table arena, or own_vals (streamed tables)
  uint64_t val_bytes = 0;
  DevBuf<uint8_t> own_vals;
};
void build_dictionary(const DeviceTable& t, uint32_t hash_bits, cudaStream_t s, uint32_t* cid_mat,
                      DictResult& out);

// Exact dictionary encoding of every column (K1 cell_scan + K2 dict_encode +
// K3 rank_sort). After encode():
//   vid[r*m+c]           rank of cell (r,c)'s value among the distinct values
//                        of column c in the escaped fragment-key order
//                        (json_escape(v) followed by '"', scoring.hpp:33-69),
//                        i.e. the fallback sort order; equal ids <=> equal bytes
//   card[c], colbase[c]  distinct count and prefix sum (host + device)
//   the per-distinct arrays below are indexed by colbase[c] + vid:
//   vlen                 segment length of the value (tokenizer + scoring)
//   count                occurrences of the value in column c
struct Encoded {
  uint64_t n = 0;
  uint32_t m = 0;
  uint64_t D = 0;  // total distinct values
  std::vector<uint64_t> card, colbase;  // host (colbase has m+1 entries)
  DevBuf<uint64_t> d_colbase;
  DevBuf<uint32_t> vid;       // n*m
  DevBuf<uint64_t> vlen;      // D
  DevBuf<uint32_t> count;     // D
  DevBuf<uint32_t> rep_row;   // D: a row holding the value
  // bytes of every distinct value (index colbase[c] + vid): the string
  // val_arena[val_off[d] .. + val_len[d]) — in the caller's table arena, or in
  // own_vals when the table was streamed from the host
  const uint8_t* val_arena = nullptr;
  uint64_t val_bytes = 0;
  DevBuf<uint64_t> val_off;   // D
  DevBuf<uint32_t> val_len;   // D
  DevBuf<uint8_t> own_vals;
  std::vector<uint64_t> total_len;  // host, per column: sum of segment lengths (stats.hpp:38)
  // host, per column (empty = none): ids of a unique column left in
  // compaction order (encode(rank_unique = false)); sorts break ties on it
  // by its escaped bytes (break_unranked_ties)
  std::vector<uint8_t> unranked;
  bool is_unranked(int c) const { return !unranked.empty() && unranked[c]; }
};

// ordered = false: ids are exact but in no particular order (equality-only
// callers: dedup, FD checks) — the escaped-order rank sort is skipped.
uint32_t debug_hash_bits();  // PO_DEBUG_HASH_BITS (abi.cu)

void encode(const DeviceTable& t, int tok, int scoring, cudaStream_t s, Encoded& e,
            uint32_t hash_bits_debug = 64, bool ordered = true, bool rank_unique = true);

// Segmented refinement sort (rank_sort / multikey_sort engine).
// Items [0, n_items) start in groups whose ids are their final start
// positions (grp_init[i]); each round sorts the unresolved items of every
// group by the next key chunk (refine_chunk_bits(grp_max) bits) (stable, so the initial item order breaks
// all remaining ties) and splits groups on chunk changes. An item is resolved
// when its run has one member or its key reports `terminal`.
// out_pos[item] receives the item's final position. grp_max must bound every
// group id of every round, i.e. the largest start position (n_items - 1).
struct RefineKey {
  // 0 = string (raw order), 1 = string (escaped order), 2 = row keys,
  // 3 = u16 symbol streams (arena holds uint16 codes >= 2, offsets count
  // symbols; end of stream = 1): token sequences of the word tokenizer
  int kind = 0;
  uint64_t skip = 0;  // string kinds: symbols [0, skip) are shared by every item
  uint32_t* item_off = nullptr;  // string kinds (set by refine_sort): symbols consumed per item
  // string keys: item i is string r = item_ref ? item_ref[i] : i, at
  // arena + str_off[r] (in symbols: bytes, or u16 codes for kind 3) of
  // str_len[r] symbols (str_len null: str_off[r + 1] - str_off[r])
  const uint8_t* arena = nullptr;
  uint64_t arena_bytes = 0;
  const uint32_t* item_ref = nullptr;
  const uint64_t* str_off = nullptr;
  const uint32_t* str_len = nullptr;
  // row keys
  uint32_t m = 0;
  const uint32_t* vid = nullptr;
  const uint64_t* colbase = nullptr;
  const uint32_t* row_leaf = nullptr;      // row -> leaf index
  const uint32_t* leaf_chunk_off = nullptr;  // leaf -> first chunk descriptor
  const uint32_t* leaf_nchunks = nullptr;
  const uint32_t* chunk_key_off = nullptr;   // chunk -> first key
  const uint32_t* chunk_nkeys = nullptr;
  const int32_t* key_field = nullptr;
  const uint8_t* key_kind = nullptr;  // unused (kept for layout); keys are vids (escaped order)
  const uint8_t* key_bits = nullptr;
  uint32_t chunk_bits = 0;       // set by refine_sort: 64 - bits(grp_max)
  uint32_t nsym0 = 0, nsym = 0;  // set by refine_sort: string symbols in round 0 / later
};

struct RefineJob {
  uint32_t n_items = 0;
  // round-0 groups: d_grp_init[i] is a group index < n_groups whose start
  // position is d_grp_start[index]; with d_grp_start == null it is the start
  // position itself. grp_max bounds every start position (n_items - 1).
  const uint32_t* d_grp_init = nullptr;
  const uint32_t* d_grp_start = nullptr;
  uint32_t n_groups = 0;
  uint32_t grp_max = 0;
  RefineKey key;
  uint32_t* d_out_pos = nullptr;
  uint32_t row_chunk_bits0 = 0;  // row keys: widest packed chunk of round 0 (0 = max)
  uint32_t row_chunk_bits = 0;   // row keys: widest packed chunk of later rounds
};

// Host-side key schedule of row sorts: keys (field, kind, bits) packed into
// chunks of at most cap0 bits (round 0) then cap bits (later rounds).
struct KeySchedule {
  std::vector<uint32_t> chunk_key_off, chunk_nkeys;
  std::vector<int32_t> key_field;
  std::vector<uint8_t> key_kind, key_bits;
  uint32_t widest0 = 1, widest = 1;
  // appends one leaf's chunks; returns its number of chunks
  uint32_t add_leaf(const std::vector<std::pair<int, uint8_t>>& keys,
                    const std::vector<uint64_t>& card, int cap0, int cap) {
    const size_t first = chunk_nkeys.size();
    bool open = false;
    int used = 0, cur_cap = 0;
    for (auto [f, kind] : keys) {
      const int b = bits_for(card[f] ? card[f] - 1 : 0);
      if (!open || used + b > cur_cap) {
        cur_cap = chunk_nkeys.size() == first ? cap0 : cap;
        chunk_key_off.push_back(uint32_t(key_field.size()));
        chunk_nkeys.push_back(0);
        used = 0;
        open = true;
      }
      key_field.push_back(f);
      key_kind.push_back(kind);
      key_bits.push_back(uint8_t(b));
      chunk_nkeys.back()++;
      used += b;
      if (chunk_nkeys.size() == first + 1) widest0 = std::max<uint32_t>(widest0, uint32_t(used));
      else widest = std::max<uint32_t>(widest, uint32_t(used));
    }
    return uint32_t(chunk_nkeys.size() - first);
  }
  void pad() {  // keep device arrays non-empty
    if (!chunk_nkeys.empty()) return;
    chunk_key_off.push_back(0);
    chunk_nkeys.push_back(0);
    key_field.push_back(0);
    key_kind.push_back(0);
    key_bits.push_back(1);
  }
};

// Several independent sorts advanced in lockstep: one host synchronisation
// per round for all of them.
void refine_sort_multi(const std::vector<RefineJob>& jobs, cudaStream_t s);

// Bits available for a key chunk next to group ids up to grp_max.
uint32_t refine_chunk_bits(uint32_t grp_max);

void refine_sort(uint32_t n_items, const uint32_t* d_grp_init, uint32_t grp_max,
                 const RefineKey& key, uint32_t* d_out_pos, cudaStream_t s,
                 uint32_t row_chunk_bits = 0);

// PHC (K9 phc_lcp): sum over entries i>=1 of hit(i) (objective.hpp:70-99).
// Schedule on device: rows[i] (u64 or u32), field orders either full
// (offsets == null, order i at fields[i*m]), CSR, or one order of m fields
// shared by every entry (uniform_order).
uint64_t phc_device(const Encoded& e, uint64_t n_entries, const uint64_t* rows64,
                    const uint32_t* rows32, const uint64_t* order_offsets,
                    const int32_t* fields, cudaStream_t s, uint64_t first_entry = 1,
                    bool uniform_order = false);

// Same over raw device arrays (vid matrix n_rows x m, per-distinct vlen).
uint64_t phc_device_raw(const uint32_t* vid, const uint64_t* vlen, const uint64_t* colbase,
                        uint64_t n_rows, uint32_t m, uint64_t n_entries, const uint64_t* rows64,
                        const uint32_t* rows32, const uint64_t* order_offsets,
                        const int32_t* fields, cudaStream_t s, uint64_t first_entry = 1,
                        bool uniform_order = false);

// The same, queued only: the sum and an out-of-range flag land in d_tot /
// d_err (both zeroed first).
void phc_device_raw_async(const uint32_t* vid, const uint64_t* vlen, const uint64_t* colbase,
                          uint64_t n_rows, uint32_t m, uint64_t n_entries, const uint64_t* rows64,
                          const uint32_t* rows32, const uint64_t* order_offsets,
                          const int32_t* fields, cudaStream_t s, unsigned long long* d_tot,
                          int* d_err, uint64_t first_entry = 1, bool uniform_order = false);

__global__ void k_invert(const uint32_t* pos, uint64_t n, uint32_t* perm);

// Stats-ranked field order (ggr.hpp:59-84) — host IEEE double, no FMA.
std::vector<int> hitcount_order(uint64_t total_rows, const std::vector<uint64_t>& card,
                                const std::vector<double>& avg, int variant);
std::vector<int> stats_order(uint64_t total_rows, const std::vector<uint64_t>& card,
                             const std::vector<double>& avg);

// Whole-table sort of all rows by escaped keys in one field order
// (sort_rows_fixed_order, objective.hpp:154-171). d_perm[pos] = row.
void sort_all_rows(const Encoded& e, const std::vector<int>& order, uint32_t* d_perm,
                   cudaStream_t s);

// The same sort as a refine job (to run in lockstep with other sorts).
// PHC of the whole table in the lexicographic order of one field order
// (first request excluded, like the fallback's phc), computed from prefix
// groups without materialising the sort.
uint64_t fixed_order_phc_device(const Encoded& e, const std::vector<int>& order, cudaStream_t s);

// Queued variant: the PHC lands in d_acc.
void fixed_order_phc_async(const Encoded& e, const std::vector<int>& order, cudaStream_t s,
                           unsigned long long* d_acc);

// True when the whole-table fallback's PHC provably cannot exceed `phc`
// (an upper bound from the dictionary counts and lengths, phc.cu).
bool fallback_cannot_win(const Encoded& e, uint64_t phc, cudaStream_t s);
// The bound queued into d_ub, and the decision from its value.
void fallback_ub_async(const Encoded& e, cudaStream_t s, double* d_ub);
bool fallback_bound_prunes(const Encoded& e, double ub, uint64_t phc);

// Leaves whose key list stops before an unranked column (Encoded::unranked):
// per leaf that column (-1: none) and the ranked key fields sorted before it
// (CSR). break_unranked_ties re-sorts every run of rows that tie on those
// keys by the column's escaped bytes (kind-1 string refine), updating pos.
struct TieSpec {
  std::vector<int32_t> tie_col;
  std::vector<uint32_t> key_off{0};
  std::vector<int32_t> key_fields;
  bool any() const {
    for (int32_t c : tie_col)
      if (c >= 0) return true;
    return false;
  }
};
// Positions of the rows of short tied runs (2..max_len rows; run[q] = start
// position of q's run, run_len[start] = its length) by the escaped bytes of
// col_of_leaf[row_leaf[row]] (distinct within a run): pos[perm[q]] = start +
// rank. One thread per position; longer runs are left alone (refine.cu).
// Bytes of cell (row, col) through its value id (Encoded's value arena).
struct CellStr {
  const uint8_t* arena;
  const uint8_t* lim;
  const uint64_t* val_off;
  const uint32_t* val_len;
  const uint32_t* vid;
  const uint64_t* colbase;
  uint32_t m;
  __device__ __forceinline__ void get(uint64_t row, uint32_t col, const uint8_t*& p,
                                      uint64_t& len) const {
    const uint64_t d = colbase[col] + vid[row * m + col];
    p = arena + val_off[d];
    len = val_len[d];
  }
};
CellStr cell_str(const Encoded& e);

void rank_short_runs(const CellStr& cs, const uint32_t* perm, const uint32_t* run,
                     const uint32_t* run_len, const uint32_t* row_leaf, const int32_t* col_of_leaf,
                     uint64_t n, uint32_t max_len, uint32_t* pos, cudaStream_t s);
// The same for the positions items[0, nt) of longer runs: 126-bit prefix
// keys, then a quadratic count per run (work = sum of squared run lengths;
// max_len = the longest run).
void rank_long_runs(const CellStr& cs, const uint32_t* perm, const uint32_t* run,
                    const uint32_t* run_len, const uint32_t* row_leaf, const int32_t* col_of_leaf,
                    const uint32_t* items, uint32_t nt, uint64_t n, uint32_t max_len, uint32_t* pos,
                    cudaStream_t s);
void break_unranked_ties(const Encoded& e, const TieSpec& ts, const uint32_t* row_leaf,
                         const uint32_t* d_leaf_off, uint32_t* pos, cudaStream_t s);

class FixedOrderSort {
 public:
  FixedOrderSort(const Encoded& e, const std::vector<int>& order, cudaStream_t s);
  const RefineJob& job() const { return job_; }
  void finish(uint32_t* d_perm);  // after the job ran: d_perm[pos] = row

 private:
  const Encoded& e_;
  TieSpec ties_;
  uint64_t n_ = 0;
  cudaStream_t s_;
  RefineJob job_;
  DevBuf<uint32_t> lco_, lnc_, cko_, cnk_, row_leaf_, grp_, pos_, start_;
  DevBuf<int32_t> kf_;
  DevBuf<uint8_t> kk_, kb_;
};

struct GgrOutput {
  uint64_t phc = 0;
  po_solve_stats stats{};
  // FD groups repeating a field pair lengthen some field orders past m
  // (ggr.hpp:280-282): the schedule's orders are then these CSR arrays
  // instead of d_orders
  bool csr = false;
  uint64_t csr_total = 0;
  DevBuf<uint64_t> csr_offsets;  // n + 1
  DevBuf<int32_t> csr_fields;    // csr_total
};

// FD checks (fd.cu): for every field pair (pa[k], pb[k]) the first row where
// their partition signatures (fd.hpp:56-64) differ (n if identical) and the
// two signatures at that row.
void fd_compare_device(const Encoded& e, const std::vector<int32_t>& pa,
                       const std::vector<int32_t>& pb, std::vector<uint64_t>& first_diff,
                       std::vector<uint64_t>& sig_a, std::vector<uint64_t>& sig_b, cudaStream_t s);

// render_prompt over a schedule (render.cu, objective.hpp:102-131): prompt i
// at out_bytes[out_off[i] .. out_off[i+1]); schedule arrays on the device.
void render_prompts_device(const DeviceTable& t, uint64_t n_entries, const uint64_t* rows,
                           const uint64_t* order_offsets, const int32_t* fields, uint64_t n_fields,
                           const std::string& system_prompt, const std::string& question,
                           DevBuf<uint64_t>& out_off, uint64_t& total,
                           const std::function<uint8_t*(uint64_t)>& dst_for, cudaStream_t s);
// dedup (cost.hpp:171-186) of the one-column table t's strings: expansion
// map and, per unique in first-occurrence order, its first index.
void dedup_device(const DeviceTable& t, uint64_t* d_expansion, uint64_t* d_unique_first,
                  uint64_t& n_unique, cudaStream_t s);

// simulate() under an unbounded cache (replay.cu, cache_sim.hpp:223-285):
// per prompt of the one-column table pt, its input tokens and raw hit (the
// longest token prefix shared with any earlier prompt); device outputs.
// The per-request report (hit, miss; d_raw becomes written) and totals.
void replay_report_device(const uint64_t* d_input, uint64_t* d_raw, uint64_t n, uint64_t min_cacheable,
                          uint64_t* d_hit, uint64_t* d_miss, unsigned long long* d_totals,
                          cudaStream_t s);
void replay_unbounded_device(const DeviceTable& pt, int tok, uint64_t* d_input, uint64_t* d_raw,
                             cudaStream_t s);

// CSV ingest (csv.cu, table.hpp:114-215): every record's cells in file order.
// Cell i = arena[cell_end[i-1] .. cell_end[i]) (cell_end[-1] = 0); record r =
// cells [rec_end_cell[r-1], rec_end_cell[r]); rec_blank: an empty unquoted
// line; unterminated: EOF inside quotes (the last record).
struct CsvParsed {
  uint64_t content_bytes = 0, n_cells = 0, n_records = 0;
  uint64_t n_closed = 0;  // records closed inside the text (a pending one follows at EOF)
  bool unterminated = false;
  DevBuf<uint8_t> arena;
  DevBuf<uint64_t> cell_end;
  DevBuf<uint64_t> rec_end, rec_line;  // [n_closed]: end cell, line after the record
  DevBuf<uint8_t> rec_blank;           // [n_closed]
  // host reads of single records (a small copy each; the per-record checks
  // run on the device: first_wrong_width)
  uint64_t end_cell(uint64_t r, cudaStream_t s) const;
  uint64_t start_line(uint64_t r, cudaStream_t s) const;
  bool blank(uint64_t r, cudaStream_t s) const;
  // first record in [1, n_records - 1) whose cell count is not h, else n_records
  uint64_t first_wrong_width(uint64_t h, cudaStream_t s) const;
};
void load_csv_device(const uint8_t* d, uint64_t len, CsvParsed& out, cudaStream_t s);

// Row-sharded solving (shard.cu). Every rank holds a
// contiguous range of the table's rows; value ids are global (escaped-order
// ranks over the whole table), the value-group tables are replicated (built
// from exchanged per-rank contributions), rows stay where they are until
// one distributed sort lays out the final schedule.
struct DistCtx {
  Comm* comm = nullptr;
  uint64_t n_global = 0;
  uint64_t row_offset = 0;  // global id of local row 0
  // global raw-byte rank of every global dense index (colbase[c] + vid):
  // built on first use (collective; every rank asks at the same point)
  std::function<const uint32_t*()> raw_ranks;
  // this rank's slice of the emitted schedule
  uint64_t slice_offset = 0, slice_count = 0;
  DevBuf<uint64_t> rows;   // slice_count global row ids
  DevBuf<int32_t> orders;  // (slice_count + 1) * m; entry i at (i + 1) * m
};

// One leaf of the final layout (DFS order): how its rows are keyed.
struct LeafKeys {
  int kind = 0;                 // 0: row id only, 1: escaped ranks of `fields`, 2: raw rank of fields[0]
  std::vector<int> fields;      // key fields in order
  std::vector<int> full_order;  // emitted field order (m fields)
};

// Distributed layout of the local rows (row_leaf[r] = leaf index) in leaf
// order, then keys, then global row id; fills dc's slice and returns the
// global PHC of the laid-out schedule (objective.hpp:94-99).
uint64_t dist_layout(DistCtx& dc, const Encoded& G, const uint32_t* d_row_leaf,
                     const std::vector<LeafKeys>& leaves, cudaStream_t s);

// GGR (ggr.hpp:144-394) on an encoded table. Writes the emitted schedule to
// d_rows (u32, n) and d_orders (i32, n*m) on the device. With `dist`, e is
// this rank's rows under global value ids and the schedule goes to dist's
// slice instead (d_rows / d_orders unused).
void ggr_device(const Encoded& e, const std::vector<std::vector<int>>& fd_groups,
                const po_ggr_config& cfg, uint32_t* d_rows, int32_t* d_orders, GgrOutput& out,
                cudaStream_t s, DistCtx* dist = nullptr);

// Row-sharded ggr(): local rows of the table in `t`, collectives over comm.
void ggr_sharded(Comm& comm, const DeviceTable& t, int tok, int scoring,
                 const std::vector<std::vector<int>>& fd_groups, const po_ggr_config& cfg,
                 DistCtx& dc, GgrOutput& out, cudaStream_t s);

}  // namespace po
