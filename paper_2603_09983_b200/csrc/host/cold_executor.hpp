// Cold-expert executor: the CPU side of the Heterogeneous Workload
// Balancer's split (§3.3, Eq. 7: T_cpu = r_c(τ)·γ·k·T_cpu_unit;
// the reference models it as miss_tokens·t_cpu_unit, sim_core.cpp:253).
// Activations whose expert is not HBM-resident this step are computed here,
// on all host cores, straight from the pinned master-copy image (the same
// tiled image the copy engine would upload), while the GPU runs the
// resident experts of the same layer; the fp32 result is added to the
// layer output by the combine kernel (y_extra).
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace moespac {

struct ColdItem {
  const uint16_t* image;  // tiled expert image (host)
  int n_tok;
  int tok[16];
  float gate[16];
};

class ColdExecutor {
 public:
  // Spin this long before sleeping (bounded by the clock, not by a pause
  // count: a pause is ~140 cycles on this pool's Xeons, so 65536 of them
  // spun ~4 ms and kept a second context's workers off the shared cores).
  // Long enough to bridge a layer's host gap (h_l D2H + wake-up).
  static constexpr long long kSpinNs = 500000;
  // layout: 1 = CUDA-core image (16-row chunks), 2 = tensor-core image (64-row chunks)
  ColdExecutor(int threads, int layout, int d, int ffn, int T);
  ~ColdExecutor();
  // y[T][d] = sum over items of gate * SwiGLU(h[tok]); h: bf16 [T][d].
  // Deterministic: fixed work partition, fixed reduction order.
  void run(const std::vector<ColdItem>& items, const uint16_t* h, float* y);
  int threads() const { return static_cast<int>(workers_.size()) + 1; }
  bool bf16_dot() const { return bf16_dot_; }
  bool pinned() const { return pin_; }

 private:
  void work(int w);
  void chunk(const ColdItem& it, int c, const float* hf, float* y, std::vector<float>& scratch) const;
  int layout_, d_, ffn_, T_, rows_;
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::atomic<int> gen_a_{0}, pending_a_{0};
  std::atomic<bool> stop_a_{false};
  // current job
  const std::vector<ColdItem>* items_ = nullptr;
  std::vector<float> hf_;                 // [T][d] fp32
  const uint16_t* hb_ = nullptr;          // [T][d] bf16 (the AVX-512 BF16 path reads it directly)
  bool bf16_dot_ = false;                 // host has VDPBF16PS (tensor-core image only)
  bool pin_ = false;                      // workers pinned one per CPU
  std::vector<std::vector<float>> part_;  // per worker [T][d]
  std::vector<std::vector<float>> scratch_;
  std::vector<std::pair<int, int>> units_;  // (item, chunk)
};

}  // namespace moespac
