// Reference-side adapter: the B200 executor behind the reference's own
// execute() signature (runtime.h:45-49). A maintainer adds this TU to the
// reference's eindecomp_core target and links libed_gpu.so.
#pragma once

#include "ed_gpu.h"
#include "eindecomp/runtime.h"

struct gpu_options_t {
  // -1: follow exec_options_t::f32 (f32 -> ED_PREC_FP32, else ED_PREC_FP64,
  // both bit-identical to the CPU executor); or force ED_PREC_BF16 / TF32.
  int precision = -1;
  int device = 0;
  // one process over several GPUs (ed_ctx_create_multi): rank r = machine % n
  // runs on devices[r]; empty = every machine on `device` as one rank. A
  // device may repeat (several ranks on one GPU: the same code path, for tests).
  vector<int> devices;
};

run_report_t execute_gpu(
  exec_graph_t const& exec,
  placement_t const& placement,
  map<int, tensor_relation_t> const& inputs,
  exec_options_t const& options = {},
  gpu_options_t const& gpu = {});
