// Outer-loop driver shared by the CP and Tucker fits (reference
// fit_common.hpp:14-53, run_outer_loop / check_finite_loss).
//
// One outer iteration is enqueued by `body`.  When `fused`, the body's first
// reconstruction pass also evaluates the objective of the model it starts
// from, so iteration k yields trace row k-1 and one standalone objective pass
// after the loop yields the last row; otherwise (extrapolation) the body ends
// with a standalone objective of the new model.  Losses land in a device
// array indexed by a device counter, so a captured CUDA graph can be replayed
// max_iters times with no host round trip when tol == 0.
//
// Semantics kept from the reference: row 0 = initial loss; stop when
// |prev - loss| / (1 + |loss|) < tol, returning the model after that
// iteration (fused mode restores a snapshot taken before the next body);
// NaN/Inf => NumericalError with the beta = 0 "data floor" message.
// time_s is the cumulative device time of the bodies (CUDA events); in fused
// mode it therefore includes the objective of the incoming model.
#pragma once
#include <functional>
#include <vector>

#include "engine.cuh"

namespace ntfg {

struct LoopHooks {
  std::function<void()> body;
  std::function<void()> objective;
  std::function<void()> snapshot;  // fused + tol > 0 only
  std::function<void()> restore;
  bool fused = true;
};

inline std::vector<ntfg_trace_row> run_fit_loop(Context& c, const ntfg_fit_config& cfg,
                                                LoopHooks& h, double* losses_dev,
                                                unsigned* flags_dev) {
  const uint64_t K = cfg.max_iters;
  const bool check_each = cfg.tol > 0.0;
  // the Python/host hook cannot run inside a graph; the native NCCL
  // communicator can (ncclAllReduce is stream-ordered and capturable)
  const bool graphs = cfg.use_graphs && (c.allreduce == nullptr || c.nccl != nullptr) && !c.profile;
  std::vector<ntfg_trace_row> trace;
  double* hl = static_cast<double*>(c.pinned.get((K + 2) * sizeof(double)));

  auto read_flags = [&]() {
    unsigned f = 0;
    NTFG_CUDA(cudaMemcpy(&f, flags_dev, sizeof(unsigned), cudaMemcpyDeviceToHost));
    raise_flags(f);
  };

  if (K == 0) {
    h.objective();
    c.sync();
    read_flags();
    double l;
    NTFG_CUDA(cudaMemcpy(&l, losses_dev, sizeof(double), cudaMemcpyDeviceToHost));
    check_finite_loss(l, cfg.beta);
    trace.push_back({0, 0.0, l});
    return trace;
  }

  auto full_body = [&]() {
    if (h.fused && check_each && h.snapshot) h.snapshot();
    h.body();
  };

  if (!h.fused) h.objective();  // row 0

  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  uint64_t per_iter_launches = 0;
  if (graphs) {
    const uint64_t before = c.stats.kernel_launches;
    NTFG_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    try {
      full_body();
    } catch (...) {
      cudaStreamEndCapture(c.stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    NTFG_CUDA(cudaStreamEndCapture(c.stream, &graph));
    NTFG_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    per_iter_launches = c.stats.kernel_launches - before;
    c.stats.kernel_launches = before;
  }

  std::vector<cudaEvent_t> ev(K + 1);
  for (auto& e : ev) NTFG_CUDA(cudaEventCreate(&e));
  auto cleanup = [&]() {
    for (auto& e : ev) cudaEventDestroy(e);
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  };

  uint64_t done = 0;        // iterations executed
  uint64_t rows = 0;        // trace rows that are final
  bool stopped = false;
  try {
    NTFG_CUDA(cudaEventRecord(ev[0], c.stream));
    for (uint64_t k = 1; k <= K; ++k) {
      if (graphs) {
        NTFG_CUDA(cudaGraphLaunch(exec, c.stream));
        c.stats.graph_launches++;
        c.stats.kernel_launches += per_iter_launches;
      } else {
        full_body();
      }
      NTFG_CUDA(cudaEventRecord(ev[k], c.stream));
      done = k;
      if (!check_each) continue;
      NTFG_CUDA(cudaEventSynchronize(ev[k]));
      // newest row known after iteration k
      const uint64_t row = h.fused ? k - 1 : k;
      NTFG_CUDA(cudaMemcpy(hl, losses_dev, (row + 1) * sizeof(double), cudaMemcpyDeviceToHost));
      read_flags();
      check_finite_loss(hl[row], cfg.beta);
      if (row >= 1 && std::abs(hl[row - 1] - hl[row]) / (1.0 + std::abs(hl[row])) < cfg.tol) {
        stopped = true;
        rows = row + 1;
        if (h.fused) h.restore();  // model after iteration `row`
        break;
      }
    }
    if (!stopped) {
      if (h.fused) h.objective();  // row K
      rows = K + 1;
    }
    c.sync();
    read_flags();
    NTFG_CUDA(cudaMemcpy(hl, losses_dev, rows * sizeof(double), cudaMemcpyDeviceToHost));
    for (uint64_t r = 0; r < rows; ++r) check_finite_loss(hl[r], cfg.beta);
    double t = 0.0;
    trace.push_back({0, 0.0, hl[0]});
    for (uint64_t r = 1; r < rows; ++r) {
      float ms = 0.f;
      if (r <= done) NTFG_CUDA(cudaEventElapsedTime(&ms, ev[r - 1], ev[r]));
      t += double(ms) * 1e-3;
      trace.push_back({r, t, hl[r]});
    }
    float total = 0.f;
    NTFG_CUDA(cudaEventElapsedTime(&total, ev[0], ev[done]));
    c.stats.device_ms = total;
    c.prof_collect();
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
  return trace;
}

}  // namespace ntfg
