/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * CPU checker for the GGR reorder + PHC path. Two libraries export this
 * interface under different prefixes:
 *   oracle/libggr_oracle.so   oracle_*  — the CPU restatement in ggr_oracle.cpp
 *   oracle/_ref/libggr_ref.so ref_*     — the reference headers themselves,
 *                                         compiled from /root/reference by
 *                                         oracle/Makefile (ref_shim.cpp)
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load them. The product path never does.
 *
 * Signatures mirror include/prefixopt_cuda.h minus the stream argument; all
 * buffers are host memory (po_table.location must be PO_LOC_HOST).
 */
#ifndef PREFIXOPT_ORACLE_H
#define PREFIXOPT_ORACLE_H

#include "../include/prefixopt_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

#define PO_ORACLE_DECLARE(prefix)                                                        \
  /* schedule in CSR form: fields of entry i at [out_order_offsets[i],         \
     out_order_offsets[i+1]); PO_ERR_SIZE when more than fields_capacity */    \
  int prefix##ggr(const po_table* t, const po_fd_groups* fds, const po_ggr_config* cfg,  \
                  int32_t tokenizer, int32_t scoring, uint64_t* out_row_ids,             \
                  uint64_t* out_order_offsets, int32_t* out_order_fields,                \
                  uint64_t fields_capacity, uint64_t* out_phc, po_solve_stats* out_stats); \
  int prefix##phc(const po_table* t, int32_t tokenizer, int32_t scoring,                \
                  uint64_t n_entries, const uint64_t* row_ids,                           \
                  const uint64_t* order_offsets, const int32_t* order_fields,            \
                  uint64_t* out_phc);                                                    \
  int prefix##sort_rows_fixed_order(const po_table* t, const int32_t* field_order,      \
                                    uint64_t* out_row_ids);                              \
  int prefix##compute_stats(const po_table* t, int32_t tokenizer, int32_t scoring,      \
                            uint64_t* out_cardinality, uint64_t* out_total_len);         \
  int prefix##fixed_order_by_hitcount_stats(uint32_t n_fields, uint64_t total_rows,     \
                                            const uint64_t* cardinality,                 \
                                            const double* avg_len, int32_t variant,      \
                                            int32_t* out_order);                         \
  int prefix##validate_fds(const po_table* t, const po_fd_groups* fds, uint8_t* out_satisfied, \
                           uint8_t* out_has_witness, uint64_t* out_row_a,                \
                           uint64_t* out_row_b, int32_t* out_agree, int32_t* out_differ); \
  int prefix##discover_fds(const po_table* t, uint64_t max_rows,                         \
                           int32_t* out_group_of_field);                                 \
  int prefix##render_prompts(const po_table* t, uint64_t n_entries, const uint64_t* row_ids, \
                             const uint64_t* order_offsets, const int32_t* order_fields,  \
                             const uint8_t* system_prompt, uint64_t system_prompt_len,    \
                             const uint8_t* question, uint64_t question_len,              \
                             uint64_t* out_offsets, uint8_t* out_bytes, uint64_t capacity, \
                             uint64_t* out_total);                                          \
  int prefix##dedup(uint64_t n, const uint8_t* arena, const uint64_t* offsets,             \
                    uint64_t* out_expansion, uint64_t* out_unique_first,                   \
                    uint64_t* out_n_unique);                                               \
  const char* prefix##last_error(void);

PO_ORACLE_DECLARE(oracle_)
PO_ORACLE_DECLARE(ref_)

#ifdef __cplusplus
}
#endif

#endif
