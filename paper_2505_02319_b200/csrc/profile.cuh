// Live per-category kernel timing with CUDA events on the launching stream.
//
// bench.py turns this on for the timed region to report the average launch
// duration of the dominant kernel group (roofline.achieved) and the time
// split of a Dyson solve; off by default (zero overhead: one branch).
#pragma once

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace pwb {

enum ProfCat {
  PROF_H = 0,    // batched H apply inside CG: plane_inv + pencil(V) + plane_fwd
  PROF_Q = 1,    // projector GEMMs (partial + reduce + apply)
  PROF_CG = 2,   // per-row CG reductions / updates
  PROF_RHS = 3,  // chi0 right-hand side (FFTs + Phi^H dV psi)
  PROF_ACC = 4,  // drho accumulation (fused inverse-x FFT + band reduction)
  PROF_NCAT = 8
};

struct Profiler {
  struct Pending {
    int cat;
    cudaEvent_t a, b;
    long long units;
  };
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<Pending> pending;
  double ms[PROF_NCAT] = {0};
  long long count[PROF_NCAT] = {0};
  long long units[PROF_NCAT] = {0};
  // per category, histogram over floor(log2(units)) (live rows of the launch group)
  static constexpr int NB = 16;
  double hms[PROF_NCAT][NB] = {};
  long long hcnt[PROF_NCAT][NB] = {};
  int rows_hint = 0;   // live rows of the running CG iteration (0 = unknown)

  cudaEvent_t take() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t begin(cudaStream_t s) {
    if (!on) return nullptr;
    cudaEvent_t e = take();
    cudaEventRecord(e, s);
    return e;
  }
  void end(int cat, cudaEvent_t a, cudaStream_t s, long long u) {
    if (!on || !a) return;
    cudaEvent_t b = take();
    cudaEventRecord(b, s);
    pending.push_back(Pending{cat, a, b, u});
  }
  // call after the stream has been synchronised
  void flush() {
    for (auto& p : pending) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, p.a, p.b) == cudaSuccess) {
        ms[p.cat] += t;
        count[p.cat] += 1;
        units[p.cat] += p.units;
        const int bkt = p.units > 0 ? std::min(NB - 1, 63 - __builtin_clzll((unsigned long long)p.units)) : 0;
        hms[p.cat][bkt] += t;
        hcnt[p.cat][bkt] += 1;
      }
      pool.push_back(p.a);
      pool.push_back(p.b);
    }
    pending.clear();
  }
  void reset() {
    pending.clear();
    for (int i = 0; i < PROF_NCAT; ++i) {
      ms[i] = 0;
      count[i] = 0;
      units[i] = 0;
      for (int b = 0; b < NB; ++b) {
        hms[i][b] = 0;
        hcnt[i][b] = 0;
      }
    }
  }
};

Profiler& prof();

}  // namespace pwb
