// ref_tool — TEST INFRASTRUCTURE ONLY (oracle). Never linked into the product.
//
// A JSON-in / JSON-out driver over the UNMODIFIED reference library
// (/root/reference/proj, built by oracle/Makefile into oracle/_ref/). It lets
// the pytest suite and the golden-fixture generator ask the reference for:
//   op=simulate      ppd::sim::run_simulation            (simulator.cpp:503-509)
//   op=generate      ppd::workload::generate_conversations (workload.cpp:90-119)
//   op=calib         CalibrationTable::defaults/to_json/hash (costmodel.cpp:220-316)
//   op=costs         full/append prefill, decode step, interference
//                                                        (costmodel.cpp:318-379)
//   op=decide        a sequence of routing::decide calls  (routing.cpp:340-387)
//   op=aggregate     metrics::aggregate over given records (metrics.cpp:79-107)
// One JSON object on stdin, one JSON object on stdout.
#include <chrono>
#include <iostream>
#include <iterator>
#include <memory>
#include <sstream>
#include <string>

#include <json.hpp>

#include "ppd/costmodel.hpp"
#include "ppd/md5.hpp"
#include "ppd/metrics.hpp"
#include "ppd/routing.hpp"
#include "ppd/simulator.hpp"
#include "ppd/workload.hpp"

using nlohmann::json;
using namespace ppd;

namespace {

cost::CalibrationTable calib_from(const json& job) {
  if (job.contains("calib_json"))
    return cost::CalibrationTable::from_json(job["calib_json"].get<std::string>());
  auto c = cost::CalibrationTable::defaults();
  if (job.contains("calib_overrides")) {
    const json& o = job["calib_overrides"];
    auto set = [&](const char* k, double& v) { if (o.contains(k)) v = o[k].get<double>(); };
    set("full_a_lin", c.full_a_lin);
    set("full_b_quad", c.full_b_quad);
    set("append_a_lin", c.append_a_lin);
    set("append_b_cross", c.append_b_cross);
    set("decode_c_base", c.decode_c_base);
    set("decode_d_batch", c.decode_d_batch);
    set("kv_bytes_per_token", c.kv_bytes_per_token);
    set("link_bandwidth", c.link_bandwidth);
    if (o.contains("prefill_service_distribution"))
      c.prefill_service_distribution = o["prefill_service_distribution"].get<std::string>();
    c.finalize();
  }
  return c;
}

workload::WorkloadSpec spec_from(const json& w) {
  workload::WorkloadSpec s;
  s.id = w.value("id", std::string("workload"));
  s.turn1 = {w.at("turn1")[0].get<long>(), w.at("turn1")[1].get<long>()};
  s.turn2plus = {w.at("turn2plus")[0].get<long>(), w.at("turn2plus")[1].get<long>()};
  s.num_turns = w.value("num_turns", 2);
  s.qps = w.value("qps", 1.0);
  s.duration_s = w.value("duration_s", 10.0);
  s.think_time_s = w.value("think_time_s", 0.0);
  s.jitter_pct = w.value("jitter_pct", 0.0);
  s.category = workload::classify(s.turn2plus);
  return s;
}

std::vector<workload::Conversation> convs_from(const json& job) {
  if (job.contains("workload"))
    return workload::generate_conversations(spec_from(job["workload"]),
                                            job.value("seed", 1ull));
  std::vector<workload::Conversation> out;
  for (const auto& c : job.at("conversations")) {
    workload::Conversation cv;
    cv.conv_id = c.at("conv_id").get<std::string>();
    cv.first_message_digest = md5(cv.conv_id);
    long ctx = 0;
    int idx = 0;
    double arrival = c.value("arrival", -1.0);
    for (const auto& t : c.at("turns")) {
      workload::TurnRequest r;
      r.conv_id = cv.conv_id;
      r.turn_index = ++idx;
      r.new_input_tokens = t[0].get<long>();
      r.target_output_tokens = t[1].get<long>();
      r.cached_context_tokens = ctx;
      r.arrival_time = idx == 1 ? arrival : -1.0;
      ctx += r.new_input_tokens + r.target_output_tokens;
      cv.turns.push_back(r);
    }
    out.push_back(std::move(cv));
  }
  return out;
}

json convs_to_json(const std::vector<workload::Conversation>& convs) {
  json arr = json::array();
  for (const auto& c : convs) {
    json turns = json::array();
    for (const auto& t : c.turns)
      turns.push_back({t.new_input_tokens, t.target_output_tokens,
                       t.cached_context_tokens, t.arrival_time});
    arr.push_back({{"conv_id", c.conv_id},
                   {"digest", digest_hex(c.first_message_digest)},
                   {"turns", turns}});
  }
  return arr;
}

routing::RoutingPolicy policy_from(const json& job) {
  if (job.value("policy", std::string("static")) == "dynamic") {
    auto t = std::make_shared<routing::DecisionTable>(
        routing::DecisionTable::from_json(job.at("table_json").get<std::string>()));
    return routing::RoutingPolicy::dynamic_policy(t);
  }
  return routing::RoutingPolicy::static_policy(job.value("x", 0.0));
}

json agg_to_json(const metrics::AggregateMetrics& a) {
  auto o = [](const std::optional<double>& v) { return v ? json(*v) : json(nullptr); };
  return {{"ttft_t1_mean", o(a.ttft_t1_mean)}, {"ttft_t1_p99", o(a.ttft_t1_p99)},
          {"ttft_t2_mean", o(a.ttft_t2_mean)}, {"ttft_t2_p99", o(a.ttft_t2_p99)},
          {"tpot_mean", o(a.tpot_mean)},       {"latency_mean", o(a.latency_mean)},
          {"tps", a.tps}, {"success_rate", a.success_rate}, {"degraded", a.degraded},
          {"total_requests", a.total_requests},
          {"completed_requests", a.completed_requests}};
}

json op_simulate(const json& job) {
  auto calib = std::make_shared<const cost::CalibrationTable>(calib_from(job));
  auto cfg = sim::ClusterConfig::from_name(job.at("cluster").get<std::string>(),
                                           policy_from(job), calib);
  if (job.contains("max_decode_batch")) cfg.max_decode_batch = job["max_decode_batch"].get<int>();
  if (job.contains("request_timeout_s")) cfg.request_timeout_s = job["request_timeout_s"].get<double>();
  auto convs = convs_from(job);
  int repeat = job.value("repeat", 1);
  sim::SimResult r;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < repeat; ++i)
    r = sim::run_simulation(cfg, convs, job.value("qps_replay", -1.0),
                            job.value("seed", 1ull), job.value("think_time_s", 0.0));
  double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::ostringstream rec;
  metrics::export_records(rec, job.value("manifest", std::string("{}")), r.records);
  json ns = json::array();
  for (const auto& n : r.node_stats)
    ns.push_back({{"role", std::string(1, n.role)}, {"prefill_busy_s", n.prefill_busy_s},
                  {"decode_busy_s", n.decode_busy_s}});
  double window = std::max(job.value("window", 0.0), r.makespan);
  return {{"records_jsonl", rec.str()},
          {"link_transfers", r.link_transfers},
          {"link_bytes", r.link_bytes},
          {"link_queue_delays", r.link_queue_delays},
          {"node_stats", ns},
          {"makespan", r.makespan},
          {"prefill_wait_samples", r.prefill_wait_samples},
          {"session_miss_fallbacks", r.session_miss_fallbacks},
          {"aggregate", agg_to_json(metrics::aggregate(r.records, window))},
          {"calib_hash", calib->hash()},
          {"wall_s", wall / repeat}};
}

json op_costs(const json& job) {
  auto c = calib_from(job);
  json out = json::array();
  for (const auto& q : job.at("queries")) {
    std::string f = q.at("f").get<std::string>();
    if (f == "full") {
      out.push_back(cost::full_prefill_time(q.at("n").get<long>(), c));
    } else if (f == "append") {
      out.push_back(cost::append_prefill_time(q.at("m").get<long>(), q.at("n").get<long>(), c));
    } else {
      cost::BatchState s;
      s.decode_batch_size = q.value("batch", 0);
      s.colocated_full_prefill_tokens = q.value("full_tokens", 0l);
      s.colocated_append_prefill_tokens = q.value("append_tokens", 0l);
      s.concurrent_prefill_ops = q.value("conc", 0);
      if (f == "interference") {
        bool clamped = false;
        double m = cost::interference_multiplier(s, c, &clamped);
        out.push_back({m, clamped});
      } else {
        out.push_back(cost::decode_step_time(s, c));
      }
    }
  }
  return {{"results", out}};
}

json op_decide(const json& job) {
  auto policy = policy_from(job);
  routing::SessionTable sessions;
  json out = json::array();
  for (const auto& q : job.at("requests")) {
    workload::TurnRequest r;
    r.turn_index = q.at("turn").get<int>();
    r.new_input_tokens = q.value("n_in", 1l);
    r.target_output_tokens = q.value("n_out", 1l);
    r.cached_context_tokens = q.value("n_ctx", 0l);
    int assign = q.value("assign", 0);
    if (q.value("evict", false)) sessions.erase(md5(q.at("conv").get<std::string>()));
    auto d = routing::decide(r, md5(q.at("conv").get<std::string>()), q.value("qps", 1.0),
                             policy, sessions, q.value("now", 0.0),
                             [assign] { return assign; });
    out.push_back({{"target", d.target == routing::RouteDecision::Target::D_local ? "D_local" : "P_path"},
                   {"x_used", d.x_used}, {"session_missing", d.session_missing},
                   {"table_miss", d.table_miss}});
  }
  return {{"decisions", out}};
}

}  // namespace

int main() {
  std::string text((std::istreambuf_iterator<char>(std::cin)), std::istreambuf_iterator<char>());
  try {
    json job = json::parse(text);
    std::string op = job.at("op").get<std::string>();
    json out;
    if (op == "simulate") out = op_simulate(job);
    else if (op == "generate") out = {{"conversations", convs_to_json(convs_from(job))}};
    else if (op == "calib") {
      auto c = calib_from(job);
      out = {{"json", c.to_json()}, {"hash", c.hash()}};
    } else if (op == "costs") out = op_costs(job);
    else if (op == "decide") out = op_decide(job);
    else throw std::invalid_argument("unknown op " + op);
    std::cout << out.dump() << "\n";
    return 0;
  } catch (const std::exception& e) {
    std::cout << json{{"error", e.what()}}.dump() << "\n";
    return 1;
  }
}
