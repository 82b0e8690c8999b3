// TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into, called by or
// shipped with the product path (paper_2410_02682_b200/, libed_gpu.so). Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
//
// A plain C++ restatement of the reference executor's arithmetic, driven by
// the same ed_plan_c the product consumes (include/ed_gpu.h). Each function
// cites the reference file:line it restates. Pinned against the compiled
// reference (oracle/_ref) and the reference's own KATs in tests/.
#pragma once
#include <stddef.h>
#include <stdint.h>

#include "../include/ed_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* kernel_eval (kernel.cc:15-68): one inner EinSum over one chunk pair, the
 * odometer over the distinct labels, first touch assigns, later touches fold
 * in odometer order; f32 rounds every operand and result through float. */
int oracle_kernel_eval(const ed_vertex_c* v, const int64_t* local_xy,
                       const double* cx, const double* cy, double* out, int f32,
                       char* err, size_t errlen);

/* eval_expr (reference.cc:3-60): the dense oracle for one expression over
 * whole tensors; bxy = concatenated input bounds. */
int oracle_eval_expr(const ed_vertex_c* v, const int64_t* bxy,
                     const double* x, const double* y, double* out,
                     char* err, size_t errlen);

/* chunk (relation.cc:31-53): out holds prod(d) chunks back to back, keys in
 * lexicographic order, each row-major over bound/d. */
void oracle_chunk(int32_t rank, const int64_t* bound, const int64_t* d,
                  const double* t, double* out);
/* assemble (relation.cc:55-78): inverse of oracle_chunk. */
void oracle_assemble(int32_t rank, const int64_t* bound, const int64_t* d,
                     const double* chunks, double* out);

/* max_rel_err (tensor.cc:9-19). */
double oracle_max_rel_err(const double* got, const double* expect, int64_t n);

/* generate_inputs (runtime.cc:552-571) for one input vertex, drawn with the
 * same libstdc++ engine and distributions. */
void oracle_generate_input(int64_t n, int32_t integer_valued, uint64_t seed,
                           int32_t vid, double* out);

/* The executor (runtime.cc:183-270, 382-451) run sequentially in exec-id
 * order (any order gives the same bits: runtime.h:8-9). inputs are whole
 * tensors per input vertex; outputs are assembled graph outputs. chunk_out,
 * when non-null, has n_exec entries (nullptr to skip) receiving each exec
 * vertex's chunk. counters: n_machines entries. */
int oracle_execute(const ed_plan_c* plan, const ed_tensor_in_c* inputs, int32_t n_inputs,
                   int32_t f32, ed_output_c* outputs, int32_t n_outputs,
                   double* const* chunk_out, ed_machine_c* counters,
                   int64_t* total_transferred, char* err, size_t errlen);

/* compute() (runtime.cc:183-270) for ONE join or refinement, given its
 * dependency chunks in dep order (used to replay a rank's schedule). */
int oracle_exec_vertex(const ed_plan_c* plan, int32_t exec_id, const double* const* deps, double* out,
                       int32_t f32, char* err, size_t errlen);

#ifdef __cplusplus
}
#endif
