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
//   op=sweep         sweep::run_sweep + results_csv, mean_over_seeds,
//                    winner_inputs/winner_distribution, compare_modes (sweep.cpp)
//   op=pareto        metrics::pareto_frontier                (metrics.cpp:109-132)
//   op=winner        metrics::winner_distribution + render   (metrics.cpp:134-225)
//   op=weight_sweep  sweep::weight_sweep                     (sweep.cpp:456-547)
//   op=plan_default  SweepPlan::full_default + to_json/hash  (sweep.cpp:44-166)
//   op=ingest_trace  workload::ingest_trace                  (workload.cpp:121-194)
//   op=gateway       a script of BackendRegistry / Gateway::route /
//                    handle_message / stats calls          (gateway.cpp:23-255)
// One JSON object on stdin, one JSON object on stdout.
#include <chrono>
#include <cmath>
#include <filesystem>
#include <optional>
#include <iostream>
#include <iterator>
#include <memory>
#include <sstream>
#include <string>

#include <json.hpp>

#include "ppd/costmodel.hpp"
#include "ppd/gateway.hpp"
#include "ppd/md5.hpp"
#include "ppd/metrics.hpp"
#include "ppd/routing.hpp"
#include "ppd/simulator.hpp"
#include "ppd/sweep.hpp"
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
  if (job.contains("trace_jsonl")) {  // real-trace replay (workload.cpp ingest_trace)
    std::istringstream in(job["trace_jsonl"].get<std::string>());
    workload::TraceFilter f;
    f.min_turns = job.value("min_turns", 2);
    f.min_turn2_input_output_ratio = job.value("min_ratio", 0.0);
    if (job.contains("sample_size")) f.sample_size = job["sample_size"].get<std::size_t>();
    f.sample_seed = job.value("sample_seed", std::uint64_t{0});
    return workload::ingest_trace(in, f);
  }
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

json gateway_item(gateway::Gateway& gw, const json& it) {
  const std::string what = it.at("do").get<std::string>();
  const double now = it.value("now", 0.0);
  try {
    if (what == "add") {
      const std::string role = it.at("role").get<std::string>();
      return {{"id", gw.registry().add(role.empty() ? '?' : role[0], it.value("address", std::string()), now)}};
    }
    if (what == "heartbeat") return {{"ok", gw.registry().heartbeat(it.at("id").get<int>(), now)}};
    if (what == "remove") return {{"removed", gw.registry().remove(it.at("id").get<int>())}};
    if (what == "invalidate") return {{"invalidated", gw.sessions().invalidate_backend(it.at("id").get<int>())}};
    if (what == "prune") return {{"removed", gw.registry().prune_dead(now, it.value("timeout", 30.0))}};
    if (what == "find") {
      auto e = gw.registry().find(it.at("id").get<int>());
      if (!e) return {{"found", false}};
      return {{"found", true}, {"role", std::string(1, e->role)}, {"address", e->address},
              {"last_heartbeat", e->last_heartbeat}};
    }
    if (what == "route") {
      gateway::RouteQuery q;
      q.conv_first_message = it.at("conv").get<std::string>();
      q.turn_index = it.at("turn").get<int>();
      q.new_input_tokens = it.value("n_in", 0L);
      q.cached_context_tokens = it.value("n_ctx", 0L);
      q.target_output_tokens = it.value("n_out", 0L);
      auto r = gw.route(q, now);
      return {{"ok", r.ok}, {"error", r.error}, {"target", r.target}, {"prefill_backend", r.prefill_backend},
              {"decode_backend", r.decode_backend}, {"x_used", r.x_used}, {"session_missing", r.session_missing},
              {"table_miss", r.table_miss}};
    }
    if (what == "message") {
      json r = json::parse(gw.handle_message(it.at("payload").get<std::string>(), now));
      r.erase("decision_latency_p99_us");
      return {{"reply", r.dump()}};
    }
    if (what == "stats") {
      auto s = gw.stats();
      return {{"queries", s.queries}, {"p_path", s.p_path}, {"d_local", s.d_local}, {"r_local", s.r_local},
              {"errors", s.errors},   {"sessions", s.sessions}, {"backends", s.backends}};
    }
  } catch (const std::invalid_argument&) {
    return {{"invalid_argument", true}};
  }
  throw std::invalid_argument("gateway script: unknown step " + what);
}

json op_gateway(const json& job) {
  gateway::Gateway gw(policy_from(job));
  gw.session_ttl_s = job.value("session_ttl_s", 3600.0);
  gw.backend_timeout_s = job.value("backend_timeout_s", 30.0);
  json out = json::array();
  for (const auto& it : job.at("script")) out.push_back(gateway_item(gw, it));
  return {{"results", out}};
}

json cell_json(const sweep::CellResult& c) { return json::parse(c.to_json()); }

json winner_json(const metrics::WinnerDistribution& d) {
  json rows = json::array();
  for (const auto& [cat, w] : d.rows) rows.push_back({cat, w.ttft_pct, w.tpot_pct, w.throughput_pct, w.avg});
  return {{"render", d.render()}, {"rows", rows}, {"cells", d.cells}, {"all_degraded_cells", d.all_degraded_cells},
          {"disagreement_fraction", d.disagreement_fraction}};
}

json nan_null(double v) { return std::isnan(v) ? json(nullptr) : json(v); }

metrics::AggregateMetrics agg_from_manifest(const json& j) {
  return sweep::CellResult::from_json(json{{"config_label", ""}, {"shape", ""}, {"x_mode", ""}, {"category", ""},
                                           {"workload_id", ""}, {"qps", 0.0}, {"seed", 0}, {"failed", false},
                                           {"metrics", j}}
                                          .dump())
      .m;
}

json op_sweep(const json& job) {
  auto plan = sweep::SweepPlan::from_json(job.at("plan").dump());
  auto calib = std::make_shared<const cost::CalibrationTable>(calib_from(job));
  std::shared_ptr<const routing::DecisionTable> table;
  if (job.contains("table_json"))
    table = std::make_shared<routing::DecisionTable>(
        routing::DecisionTable::from_json(job["table_json"].get<std::string>()));
  std::optional<std::filesystem::path> manifest;
  if (job.contains("manifest_dir")) manifest = job["manifest_dir"].get<std::string>();
  auto rs = sweep::run_sweep(plan, calib, job.value("parallelism", 1), manifest, table);
  json cells = json::array();
  for (const auto& c : rs.cells) cells.push_back(cell_json(c));
  json means = json::array();
  for (const auto& [key, m] : sweep::mean_over_seeds(rs)) {
    sweep::CellResult holder;
    holder.m = m;
    means.push_back({std::get<0>(key), std::get<1>(key), std::get<2>(key), cell_json(holder)["metrics"]});
  }
  json out{{"plan_hash", rs.plan_hash}, {"calibration_hash", rs.calibration_hash}, {"cells", cells},
           {"csv", sweep::results_csv(rs)}, {"means", means}};
  try {
    out["winner"] = winner_json(metrics::winner_distribution(sweep::winner_inputs(rs)));
  } catch (const std::invalid_argument& e) {
    out["winner"] = {{"error", e.what()}};
  }
  json cmp = json::object();
  for (const auto& c : job.value("compare", json::array())) {
    json rows = json::array();
    for (const auto& r : sweep::compare_modes(rs, c[0].get<std::string>(), c[1].get<std::string>(),
                                              c[2].get<std::string>()))
      rows.push_back({r.shape, nan_null(r.low), nan_null(r.med), nan_null(r.high), r.low_n, r.med_n, r.high_n});
    cmp[c[0].get<std::string>() + "|" + c[1].get<std::string>() + "|" + c[2].get<std::string>()] = rows;
  }
  out["compare"] = cmp;
  return out;
}

json op_pareto(const json& job) {
  std::vector<metrics::ParetoPoint> pts;
  for (const auto& p : job.at("points")) pts.push_back({p[0].get<double>(), p[1].get<double>(), p[2].get<std::string>()});
  json f = json::array();
  for (const auto& p : metrics::pareto_frontier(pts)) f.push_back({p.ttft_p99, p.tps, p.label});
  return {{"frontier", f}};
}

json op_winner(const json& job) {
  std::vector<metrics::WinnerCell> cells;
  for (const auto& c : job.at("cells")) {
    metrics::WinnerCell w;
    w.workload_id = c.at("workload_id").get<std::string>();
    w.qps = c.at("qps").get<double>();
    w.config_label = c.at("config_label").get<std::string>();
    w.category = c.at("category").get<std::string>();
    w.m = agg_from_manifest(c.at("metrics"));
    cells.push_back(w);
  }
  return winner_json(metrics::winner_distribution(cells));
}

json op_weight_sweep(const json& job) {
  auto calib = std::make_shared<const cost::CalibrationTable>(calib_from(job));
  auto tmp = sweep::SweepPlan::from_json(json{{"configs", json::array()}, {"workloads", json::array({job.at("base")})},
                                              {"qps_levels", json::array()}, {"seeds", json::array()},
                                              {"duration_s", 0.0}}
                                             .dump());
  std::vector<routing::GridSpec> grid = routing::default_grid();
  if (job.contains("grid_keys")) {
    std::vector<routing::GridSpec> sub;
    for (const auto& k : job["grid_keys"])
      for (const auto& g : grid)
        if (g.key.str() == k.get<std::string>()) sub.push_back(g);
    grid = sub;
  }
  json rows = json::array();
  for (const auto& r : sweep::weight_sweep(job.at("shape").get<std::string>(), tmp.workloads.at(0),
                                           job.at("qps_levels").get<std::vector<double>>(),
                                           job.at("w_tpot_list").get<std::vector<double>>(), calib, grid,
                                           job.at("seeds").get<std::vector<std::uint64_t>>()))
    rows.push_back({r.w_tpot, nan_null(r.ttft_change), nan_null(r.tpot_change), r.d_local_ratio});
  return {{"rows", rows}};
}

json op_plan_default() {
  auto p = sweep::SweepPlan::full_default();
  return {{"plan_json", p.to_json()}, {"hash", p.hash()}, {"cell_count", p.cell_count()}};
}

json op_ingest_trace(const json& job) {
  std::istringstream in(job.at("trace_jsonl").get<std::string>());
  workload::TraceFilter f;
  f.min_turns = job.value("min_turns", 2);
  f.min_turn2_input_output_ratio = job.value("min_ratio", 0.0);
  if (job.contains("sample_size")) f.sample_size = job["sample_size"].get<std::size_t>();
  f.sample_seed = job.value("sample_seed", 0ull);
  json convs = json::array();
  for (const auto& c : workload::ingest_trace(in, f)) {
    json turns = json::array();
    for (const auto& t : c.turns) turns.push_back({t.new_input_tokens, t.target_output_tokens, t.cached_context_tokens});
    convs.push_back({{"conv_id", c.conv_id}, {"turns", turns}});
  }
  return {{"conversations", convs}};
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
    else if (op == "sweep") out = op_sweep(job);
    else if (op == "pareto") out = op_pareto(job);
    else if (op == "winner") out = op_winner(job);
    else if (op == "weight_sweep") out = op_weight_sweep(job);
    else if (op == "plan_default") out = op_plan_default();
    else if (op == "ingest_trace") out = op_ingest_trace(job);
    else if (op == "gateway") out = op_gateway(job);
    else throw std::invalid_argument("unknown op " + op);
    std::cout << out.dump() << "\n";
    return 0;
  } catch (const std::exception& e) {
    std::cout << json{{"error", e.what()}}.dump() << "\n";
    return 1;
  }
}
