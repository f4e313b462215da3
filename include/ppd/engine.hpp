// ppd/engine.hpp — the DEVICE clock: the same P/D/R node layout, router,
// sessions and KV-manager semantics as run_simulation (simulator.hpp), but
// every prefill, decode iteration and P->D KV hop executes on B200s through
// the C-ABI (include/ppd_b200.h) and the engine's clock advances by the
// measured CUDA-event durations.
//
// Node iteration (B200 design): one ppd_step per iteration =
// all running decode rows + the next chunk (<= prefill_chunk tokens) of the
// node's active prefill job (append chunks ride inside the decode step, the
// PPD argument). P nodes run prefill chunks only. When a P job finishes, the
// tokens the decode node is missing (need = ctx + new - have, reference
// simulator.cpp:349-353) are copied P pool -> D pool (ppd_kv_copy, NVLink when
// the nodes sit on different GPUs). First token = the token sampled from the
// prefill's last row (local) or its arrival on D (P path); at completion the
// last sampled token's KV is written by a KV-only row so the node's cache
// covers exactly ctx + new + output tokens (= reference prefix_cache, :428).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ppd/costmodel.hpp"
#include "ppd/routing.hpp"
#include "ppd/simulator.hpp"

namespace ppd::engine {

struct ModelShape {
  std::string name = "tiny";  // tiny | llama8b | qwen32b
  int n_layers = 0;           // 0 = the shape's own
};

struct DeviceOptions {
  ModelShape model;
  std::uint64_t weight_seed = 1;
  std::uint64_t token_seed = 1;
  std::vector<int> gpus = {0};   // node i runs on gpus[i % gpus.size()]
  int kv_blocks_per_node = 0;    // 0: sized from the trace
  int prefill_chunk = 2048;      // prefill tokens per iteration (D / R nodes: rides with decode rows)
  int p_prefill_chunk = 8192;    // P nodes (prefill only): tokens per iteration
  int max_step_tokens = 0;       // 0: prefill_chunk + max_decode_batch + 64
  bool record_steps = false;     // emit the step log (oracle replay)
  bool record_tokens = true;     // emit generated token ids per request
  bool realtime = false;         // wall-clock run: a worker thread per node, asynchronous KV hops
  static DeviceOptions from_json(const std::string& text);
};

struct DeviceRun {
  sim::SimResult sim;
  std::string device_json;  // per-node / per-link device stats, tokens, step log
};

DeviceRun run_on_device(const sim::ClusterConfig& cfg, const std::vector<workload::Conversation>& convs,
                        double qps_replay, std::uint64_t seed, double think_time_s, const DeviceOptions& opt);

// Phase 1 of Algorithm 1 on the device: a BenchmarkRunner that runs each grid
// workload through run_on_device with x=0 / x=1 and returns the device-clock
// (mean turn-2+ TTFT, mean TPOT).
routing::BenchmarkRunner device_benchmark_runner(const std::string& cluster, const DeviceOptions& opt,
                                                 std::shared_ptr<const cost::CalibrationTable> calib,
                                                 std::vector<std::uint64_t> seeds);

}  // namespace ppd::engine
