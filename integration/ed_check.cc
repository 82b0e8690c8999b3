// Parity driver (test infrastructure): the reference's run_end_to_end flow
// (runtime.cc:518-550) with execute() and execute_gpu() side by side on the
// same plan and inputs. Usage: ed_check <graphs dir> [precision]
#include <cstdio>
#include <cstdlib>

#include <algorithm>

#include <cuda_runtime.h>

#include "eindecomp/parse.h"
#include "execute_gpu.h"

int main(int argc, char** argv) {
  string dir = argc > 1 ? argv[1] : "/root/reference/proj/graphs";
  int prec = argc > 2 ? std::atoi(argv[2]) : -1;
  int failed = 0, ran = 0;
  for(string name: {"matmul.eg", "ffnn.eg", "softmax.eg", "attention.eg"}) {
    eingraph_t g;
    try {
      g = parse_eingraph_file(dir + "/" + name);
    } catch(std::exception const& e) {
      std::printf("SKIP %s (%s)\n", name.c_str(), e.what());
      continue;
    }
    for(int64_t p: {1, 4, 8}) {
      for(int64_t l: {1, 2, 4}) {
        auto inputs = generate_inputs(g, uint64_t(1000 + p * 10 + l));
        auto pipe = build_pipeline(g, p, l, 0.01);
        map<int, tensor_relation_t> chunked;
        for(auto const& [vid, t]: inputs) chunked.insert({vid, chunk(t, pipe.tg.d[vid])});
        for(int variant = 0; variant != 3; ++variant) {
          // f64 and f32 in the reference's default round-robin mode, f64 threaded
          const bool f32 = variant == 1;
          exec_options_t opt;
          opt.f32 = f32;
          opt.mode = variant == 2 ? sched_mode_t::threaded : sched_mode_t::round_robin;
          auto cpu = execute(pipe.exec, pipe.placement, chunked, opt);
          // one rank on device 0, and (L > 1) L ranks driven by this one
          // process over the devices present (cycled: ranks share a device
          // when there are fewer GPUs than machines)
          for(int multi = 0; multi != (l > 1 ? 2 : 1); ++multi) {
          gpu_options_t go;
          go.precision = prec;
          if(multi) {
            int ndev = 1;
            cudaGetDeviceCount(&ndev);
            for(int64_t r = 0; r != l; ++r) go.devices.push_back(int(r % std::max(1, ndev)));
          }
          auto gpu = execute_gpu(pipe.exec, pipe.placement, chunked, opt, go);
          double err = 0.0;
          bool same = true;
          for(auto const& [vid, t]: cpu.outputs) {
            same = same && (t == gpu.outputs.at(vid));
            err = std::max(err, max_rel_err(gpu.outputs.at(vid), t));
          }
          bool counters = cpu.total_transferred == gpu.total_transferred && cpu.max_site_cost == gpu.max_site_cost &&
                          cpu.wall_steps == gpu.wall_steps;
          for(size_t m = 0; m != cpu.machines.size(); ++m) {
            counters = counters && cpu.machines[m].fp == gpu.machines[m].fp &&
                       cpu.machines[m].sent == gpu.machines[m].sent &&
                       cpu.machines[m].received == gpu.machines[m].received;
          }
          bool audit = audit_violations(gpu, pipe.exec).empty();
          // exp included: the device runs the host libm's algorithm (csrc/libm_exp.cuh)
          bool ok = counters && audit && same;
          ++ran;
          failed += !ok;
          std::printf("%s %s p=%lld L=%lld %s%s%s exact=%d max_rel_err=%.3e counters=%d audit=%d wall_steps=%lld\n",
                      ok ? "PASS" : "FAIL", name.c_str(), (long long)p, (long long)l, f32 ? "f32" : "f64",
                      variant == 2 ? " threaded" : "", multi ? " ranks=L" : "", int(same), err, int(counters),
                      int(audit), (long long)gpu.wall_steps);
          }
        }
      }
    }
  }
  std::printf("%d/%d passed\n", ran - failed, ran);
  return failed ? 1 : 0;
}
