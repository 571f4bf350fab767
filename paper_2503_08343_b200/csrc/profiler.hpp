// Optional per-kernel-class timing with CUDA events on the launching stream,
// plus the ALGORITHMIC flops / bytes of each launch, for the roofline fields
// of bench.py. Off by default (zero overhead: the launch runs directly).
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <string>
#include <vector>

namespace gmrf {

struct KernelStat {
  long long launches = 0;
  double ms = 0.0, flops = 0.0, bytes = 0.0;
};

class KernelProfiler {
 public:
  bool on = false;
  bool level_detail = false;  // suffix kernel classes with "@<level>"

  std::string tag(const char* base, int level) const {
    return level_detail ? std::string(base) + "@" + std::to_string(level) : std::string(base);
  }

  template <typename F>
  void run(cudaStream_t s, const std::string& name, double flops, double bytes, F&& launch) {
    if (!on) {
      launch();
      return;
    }
    cudaEvent_t a = take(), b = take();
    cudaEventRecord(a, s);
    launch();
    cudaEventRecord(b, s);
    pending_.push_back({name, a, b, flops, bytes});
  }

  void flush() {
    for (auto& p : pending_) {
      cudaEventSynchronize(p.b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, p.a, p.b);
      KernelStat& k = stats[p.name];
      k.launches += 1;
      k.ms += ms;
      k.flops += p.flops;
      k.bytes += p.bytes;
      pool_.push_back(p.a);
      pool_.push_back(p.b);
    }
    pending_.clear();
  }

  void reset() {
    flush();
    stats.clear();
  }

  ~KernelProfiler() {
    flush();
    for (cudaEvent_t e : pool_) cudaEventDestroy(e);
  }

  std::map<std::string, KernelStat> stats;

 private:
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
    double flops, bytes;
  };
  cudaEvent_t take() {
    if (pool_.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool_.back();
    pool_.pop_back();
    return e;
  }
  std::vector<Pending> pending_;
  std::vector<cudaEvent_t> pool_;
};

}  // namespace gmrf
