// capi.cpp — JSON front door of the engine (include/ppd_engine.h).
#include <chrono>
#include <cmath>
#include <filesystem>
#include <optional>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <thread>

#include <json.hpp>

#include "../../include/ppd_engine.h"
#include "ppd/costmodel.hpp"
#include "ppd/engine.hpp"
#include "ppd/gateway.hpp"
#include "ppd/kvcache.hpp"
#include "ppd/md5.hpp"
#include "ppd/metrics.hpp"
#include "ppd/routing.hpp"
#include "ppd/simulator.hpp"
#include "ppd/sweep.hpp"
#include "ppd/workload.hpp"

using nlohmann::json;
using namespace ppd;

namespace {

thread_local std::string g_err;

cost::CalibrationTable calib_from(const json& job) {
  if (job.contains("calib_json")) return cost::CalibrationTable::from_json(job["calib_json"].get<std::string>());
  cost::CalibrationTable c = cost::CalibrationTable::defaults();
  if (job.contains("calib_overrides")) {
    const json& o = job["calib_overrides"];
    const std::pair<const char*, double*> fields[] = {
        {"full_a_lin", &c.full_a_lin},         {"full_b_quad", &c.full_b_quad},
        {"append_a_lin", &c.append_a_lin},     {"append_b_cross", &c.append_b_cross},
        {"decode_c_base", &c.decode_c_base},   {"decode_d_batch", &c.decode_d_batch},
        {"kv_bytes_per_token", &c.kv_bytes_per_token}, {"link_bandwidth", &c.link_bandwidth}};
    for (const auto& [k, dst] : fields)
      if (o.contains(k)) *dst = o[k].get<double>();
    if (o.contains("prefill_service_distribution"))
      c.prefill_service_distribution = o["prefill_service_distribution"].get<std::string>();
    c.finalize();
  }
  return c;
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
  if (job.contains("workload")) {
    const json& w = job["workload"];
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
    return workload::generate_conversations(s, job.value("seed", std::uint64_t{1}));
  }
  std::vector<workload::Conversation> out;
  for (const json& c : job.at("conversations")) {
    workload::Conversation cv;
    cv.conv_id = c.at("conv_id").get<std::string>();
    cv.first_message_digest = md5(cv.conv_id);
    long ctx = 0;
    const double arrival = c.value("arrival", -1.0);
    for (const json& t : c.at("turns")) {
      workload::TurnRequest r;
      r.conv_id = cv.conv_id;
      r.turn_index = int(cv.turns.size()) + 1;
      r.new_input_tokens = t[0].get<long>();
      r.target_output_tokens = t[1].get<long>();
      r.cached_context_tokens = ctx;
      r.arrival_time = r.turn_index == 1 ? arrival : -1.0;
      ctx += r.new_input_tokens + r.target_output_tokens;
      cv.turns.push_back(r);
    }
    out.push_back(std::move(cv));
  }
  return out;
}

routing::RoutingPolicy policy_from(const json& job) {
  if (job.value("policy", std::string("static")) == "dynamic") {
    auto t = std::make_shared<routing::DecisionTable>(
        routing::DecisionTable::from_json(job.at("table_json").get<std::string>()));
    return routing::RoutingPolicy::dynamic_policy(t);
  }
  return routing::RoutingPolicy::static_policy(job.value("x", 0.0));
}

json agg_json(const metrics::AggregateMetrics& a) {
  auto o = [](const std::optional<double>& v) { return v ? json(*v) : json(nullptr); };
  return {{"ttft_t1_mean", o(a.ttft_t1_mean)}, {"ttft_t1_p99", o(a.ttft_t1_p99)},
          {"ttft_t2_mean", o(a.ttft_t2_mean)}, {"ttft_t2_p99", o(a.ttft_t2_p99)},
          {"tpot_mean", o(a.tpot_mean)},       {"latency_mean", o(a.latency_mean)},
          {"tps", a.tps},                      {"success_rate", a.success_rate},
          {"degraded", a.degraded},            {"total_requests", a.total_requests},
          {"completed_requests", a.completed_requests},
          {"ttft_t1_p50", o(a.ttft_t1_p50)},   {"ttft_t2_p50", o(a.ttft_t2_p50)},
          {"tpot_p50", o(a.tpot_p50)},         {"tpot_p99", o(a.tpot_p99)}};
}

json result_json(const sim::SimResult& r, const json& job, const std::string& calib_hash, double wall) {
  std::ostringstream rec;
  metrics::export_records(rec, job.value("manifest", std::string("{}")), r.records);
  json ns = json::array();
  for (const sim::NodeStats& n : r.node_stats)
    ns.push_back({{"role", std::string(1, n.role)}, {"prefill_busy_s", n.prefill_busy_s},
                  {"decode_busy_s", n.decode_busy_s}});
  json kv = json::array();
  for (const sim::KvTableSnapshot& t : r.kv_tables)
    kv.push_back({{"node", t.node}, {"conv_id", t.conv_id}, {"tokens", t.tokens}, {"blocks", t.blocks}});
  const double window = std::max(job.value("window", 0.0), r.makespan);
  return {{"records_jsonl", rec.str()},
          {"link_transfers", r.link_transfers},
          {"link_bytes", r.link_bytes},
          {"link_queue_delays", r.link_queue_delays},
          {"node_stats", ns},
          {"makespan", r.makespan},
          {"prefill_wait_samples", r.prefill_wait_samples},
          {"session_miss_fallbacks", r.session_miss_fallbacks},
          {"aggregate", agg_json(metrics::aggregate(r.records, window))},
          {"kv_tables", kv},
          {"route_decisions", r.route_decisions},
          {"calib_hash", calib_hash},
          {"wall_s", wall}};
}

// op=fit_calibration: device samples -> CalibrationTable (costmodel.hpp fit_from_measurements)
std::string fit(const json& job) {
  cost::DeviceSamples s;
  const json& j = job.at("samples");
  for (const json& r : j.value("full", json::array())) s.full.emplace_back(r[0].get<long>(), r[1].get<double>());
  for (const json& r : j.value("append", json::array()))
    s.append.emplace_back(r[0].get<long>(), r[1].get<long>(), r[2].get<double>());
  for (const json& r : j.value("decode", json::array())) s.decode.emplace_back(r[0].get<int>(), r[1].get<double>());
  for (const json& r : j.value("interference", json::array()))
    s.interference.push_back({cost::prefill_kind_from_string(r.at("kind").get<std::string>()),
                              r.at("prefill_tokens").get<long>(), r.at("concurrent_prefills").get<int>(),
                              r.at("decode_batch").get<int>(), r.at("tpot_multiplier").get<double>()});
  s.kv_bytes_per_token = j.value("kv_bytes_per_token", 0.0);
  s.link_bandwidth = j.value("link_bandwidth", 0.0);
  const cost::CalibrationTable c = cost::fit_from_measurements(s);
  return json{{"calib_json", c.to_json()}, {"hash", c.hash()}}.dump();
}

// op=build_table: Phase 1 of Algorithm 1 (routing.cpp:220-244) over the default
// 90-key grid with a virtual-clock runner on the given (e.g. device-fitted)
// calibration -> the decision table the dynamic router consumes.
std::string build_table(const json& job) {
  auto calib = std::make_shared<const cost::CalibrationTable>(calib_from(job));
  const std::string cluster = job.value("cluster", std::string("1P_3D"));
  std::vector<std::uint64_t> seeds = job.value("seeds", std::vector<std::uint64_t>{1});
  const double duration = job.value("duration_s", 10.0);
  routing::BenchmarkRunner runner = [&](const routing::GridSpec& g, int x) -> std::optional<std::pair<double, double>> {
    double ttft = 0, tpot = 0;
    int n = 0;
    for (std::uint64_t seed : seeds) {
      workload::WorkloadSpec spec = g.spec;
      spec.duration_s = duration;
      const auto convs = workload::generate_conversations(spec, seed);
      auto cfg = sim::ClusterConfig::from_name(cluster, routing::RoutingPolicy::static_policy(double(x)), calib);
      const sim::SimResult r = sim::run_simulation(cfg, convs, -1, seed);
      const auto a = metrics::aggregate(r.records, std::max(spec.duration_s, r.makespan));
      if (!a.ttft_t2_mean || !a.tpot_mean) return std::nullopt;
      ttft += *a.ttft_t2_mean;
      tpot += *a.tpot_mean;
      ++n;
    }
    if (n == 0) return std::nullopt;
    return std::make_pair(ttft / n, tpot / n);
  };
  if (job.value("clock", std::string("virtual")) == "device") {
    // Phase 1 on the B200s: every (grid key, x) cell runs through the engine's
    // device clock (engine::device_benchmark_runner)
    const engine::DeviceOptions opt = engine::DeviceOptions::from_json(job.value("device", json::object()).dump());
    const routing::BenchmarkRunner dev = engine::device_benchmark_runner(cluster, opt, calib, seeds);
    runner = [dev, duration](const routing::GridSpec& g, int x) {
      routing::GridSpec h = g;
      h.spec.duration_s = duration;
      return dev(h, x);
    };
  }
  std::vector<routing::GridSpec> grid = routing::default_grid();
  if (job.contains("grid_keys")) {  // a subset of the 90 keys (absent keys route x = 0, routing.cpp:233-240)
    const auto keys = job["grid_keys"].get<std::vector<std::string>>();
    std::erase_if(grid, [&](const routing::GridSpec& g) {
      return std::find(keys.begin(), keys.end(), g.key.str()) == keys.end();
    });
  }
  routing::SLOWeights w{job.value("w_ttft", 1.0), job.value("w_tpot", 1.0)};
  const routing::DecisionTable t = routing::build_decision_table(grid, w, runner, calib->hash());
  return json{{"table_json", t.to_json()}, {"calib_hash", calib->hash()}, {"grid_keys", grid.size()}}.dump();
}

// ---- §8f-2 / §8f-4: sweep harness, analyses, trace ingest -----------------
json cell_json(const sweep::CellResult& c) { return json::parse(c.to_json()); }

metrics::AggregateMetrics agg_from(const json& j) {
  // the manifest format (reference fields); missing optionals stay empty
  sweep::CellResult c = sweep::CellResult::from_json(
      json{{"config_label", ""}, {"shape", ""}, {"x_mode", ""}, {"category", ""}, {"workload_id", ""},
           {"qps", 0.0}, {"seed", 0}, {"failed", false}, {"metrics", j}}
          .dump());
  return c.m;
}

json winner_json(const metrics::WinnerDistribution& d) {
  json rows = json::array();
  for (const auto& [cat, w] : d.rows) rows.push_back({cat, w.ttft_pct, w.tpot_pct, w.throughput_pct, w.avg});
  return {{"render", d.render()}, {"rows", rows}, {"cells", d.cells}, {"all_degraded_cells", d.all_degraded_cells},
          {"disagreement_fraction", d.disagreement_fraction}};
}

json nan_null(double v) { return std::isnan(v) ? json(nullptr) : json(v); }

// op=sweep: run a SweepPlan (reference plan JSON) on the virtual clock or, with
// "clock": "device", every cell on the GPUs; returns cells, CSV, seed means,
// the winner distribution and the requested mode comparisons.
std::string op_sweep(const json& job) {
  const sweep::SweepPlan plan = sweep::SweepPlan::from_json(job.at("plan").dump());
  auto calib = std::make_shared<const cost::CalibrationTable>(calib_from(job));
  std::shared_ptr<const routing::DecisionTable> table;
  if (job.contains("table_json"))
    table = std::make_shared<routing::DecisionTable>(
        routing::DecisionTable::from_json(job["table_json"].get<std::string>()));
  std::optional<std::filesystem::path> manifest;
  if (job.contains("manifest_dir")) manifest = job["manifest_dir"].get<std::string>();
  const auto t0 = std::chrono::steady_clock::now();
  sweep::ResultSet rs;
  if (job.value("clock", std::string("virtual")) == "device") {
    const engine::DeviceOptions opt = engine::DeviceOptions::from_json(job.value("device", json::object()).dump());
    rs = sweep::run_sweep_on_device(plan, calib, opt, manifest, table);
  } else {
    rs = sweep::run_sweep(plan, calib, job.value("parallelism", 1), manifest, table);
  }
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  json cells = json::array();
  for (const auto& c : rs.cells) cells.push_back(cell_json(c));
  json means = json::array();
  for (const auto& [key, m] : sweep::mean_over_seeds(rs))
  {
    sweep::CellResult holder;
    holder.m = m;
    means.push_back({std::get<0>(key), std::get<1>(key), std::get<2>(key), cell_json(holder)["metrics"]});
  }
  json out{{"plan_hash", rs.plan_hash}, {"calibration_hash", rs.calibration_hash}, {"cells", cells},
           {"csv", sweep::results_csv(rs)}, {"means", means}, {"wall_s", wall}};
  try {
    out["winner"] = winner_json(metrics::winner_distribution(sweep::winner_inputs(rs)));
  } catch (const std::invalid_argument& e) {
    out["winner"] = {{"error", e.what()}};
  }
  json cmp = json::object();
  for (const json& c : job.value("compare", json::array())) {
    json rows = json::array();
    for (const auto& r : sweep::compare_modes(rs, c[0].get<std::string>(), c[1].get<std::string>(),
                                              c[2].get<std::string>()))
      rows.push_back({r.shape, nan_null(r.low), nan_null(r.med), nan_null(r.high), r.low_n, r.med_n, r.high_n});
    cmp[c[0].get<std::string>() + "|" + c[1].get<std::string>() + "|" + c[2].get<std::string>()] = rows;
  }
  out["compare"] = cmp;
  return out.dump();
}

std::string op_pareto(const json& job) {
  std::vector<metrics::ParetoPoint> pts;
  for (const json& p : job.at("points")) pts.push_back({p[0].get<double>(), p[1].get<double>(), p[2].get<std::string>()});
  json f = json::array();
  for (const auto& p : metrics::pareto_frontier(pts)) f.push_back({p.ttft_p99, p.tps, p.label});
  return json{{"frontier", f}}.dump();
}

std::string op_winner(const json& job) {
  std::vector<metrics::WinnerCell> cells;
  for (const json& c : job.at("cells"))
    cells.push_back({c.at("workload_id").get<std::string>(), c.at("qps").get<double>(),
                     c.at("config_label").get<std::string>(), c.at("category").get<std::string>(),
                     agg_from(c.at("metrics"))});
  return winner_json(metrics::winner_distribution(cells)).dump();
}

std::vector<routing::GridSpec> grid_from(const json& job) {
  std::vector<routing::GridSpec> grid = routing::default_grid();
  if (job.contains("grid_keys")) {  // subset of the default grid by key string
    std::vector<routing::GridSpec> sub;
    for (const json& k : job["grid_keys"])
      for (const auto& g : grid)
        if (g.key.str() == k.get<std::string>()) sub.push_back(g);
    grid = sub;
  }
  return grid;
}

std::string op_weight_sweep(const json& job) {
  auto calib = std::make_shared<const cost::CalibrationTable>(calib_from(job));
  sweep::SweepPlan tmp = sweep::SweepPlan::from_json(
      json{{"configs", json::array()}, {"workloads", json::array({job.at("base")})}, {"qps_levels", json::array()},
           {"seeds", json::array()}, {"duration_s", 0.0}}
          .dump());
  json rows = json::array();
  for (const auto& r : sweep::weight_sweep(job.at("shape").get<std::string>(), tmp.workloads.at(0),
                                           job.at("qps_levels").get<std::vector<double>>(),
                                           job.at("w_tpot_list").get<std::vector<double>>(), calib, grid_from(job),
                                           job.at("seeds").get<std::vector<std::uint64_t>>()))
    rows.push_back({r.w_tpot, nan_null(r.ttft_change), nan_null(r.tpot_change), r.d_local_ratio});
  return json{{"rows", rows}}.dump();
}

std::string op_plan_default() {
  const sweep::SweepPlan p = sweep::SweepPlan::full_default();
  return json{{"plan_json", p.to_json()}, {"hash", p.hash()}, {"cell_count", p.cell_count()}}.dump();
}

std::string op_ingest_trace(const json& job) {
  std::istringstream in(job.at("trace_jsonl").get<std::string>());
  workload::TraceFilter f;
  f.min_turns = job.value("min_turns", 2);
  f.min_turn2_input_output_ratio = job.value("min_ratio", 0.0);
  if (job.contains("sample_size")) f.sample_size = job["sample_size"].get<std::size_t>();
  f.sample_seed = job.value("sample_seed", std::uint64_t{0});
  json convs = json::array();
  for (const auto& c : workload::ingest_trace(in, f)) {
    json turns = json::array();
    for (const auto& t : c.turns)
      turns.push_back({t.new_input_tokens, t.target_output_tokens, t.cached_context_tokens});
    convs.push_back({{"conv_id", c.conv_id}, {"turns", turns}});
  }
  return json{{"conversations", convs}}.dump();
}

// ---- gateway ----------------------------------------------
// op=gateway: a script of registry / route / wire-message calls against one
// in-process Gateway with an explicit clock; oracle/ref_tool.cpp runs the same
// script through the reference gateway (parity test: tests/test_gateway.py).
json gateway_item(gateway::Gateway& gw, const json& it) {
  const std::string what = it.at("do").get<std::string>();
  const double now = it.value("now", 0.0);
  try {
    if (what == "add") {
      const std::string role = it.at("role").get<std::string>();
      return {{"id", gw.registry().add(role.empty() ? '?' : role[0], it.value("address", std::string()), now,
                                        it.value("gpu", -1))}};
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
      const gateway::RouteReply r = gw.route(q, now);
      json o = {{"ok", r.ok}, {"error", r.error}, {"target", r.target}, {"prefill_backend", r.prefill_backend},
                {"decode_backend", r.decode_backend}, {"x_used", r.x_used}, {"session_missing", r.session_missing},
                {"table_miss", r.table_miss}};
      if (r.decode_gpu >= 0) o["decode_gpu"] = r.decode_gpu;
      if (r.prefill_gpu >= 0) o["prefill_gpu"] = r.prefill_gpu;
      return o;
    }
    if (what == "message") {
      json r = json::parse(gw.handle_message(it.at("payload").get<std::string>(), now));
      r.erase("decision_latency_p99_us");  // wall-clock measurement, not comparable
      return {{"reply", r.dump()}};
    }
    if (what == "stats") {
      const gateway::GatewayStats s = gw.stats();
      return {{"queries", s.queries}, {"p_path", s.p_path}, {"d_local", s.d_local}, {"r_local", s.r_local},
              {"errors", s.errors},   {"sessions", s.sessions}, {"backends", s.backends}};
    }
  } catch (const std::invalid_argument& e) {
    return {{"invalid_argument", true}};
  }
  throw std::invalid_argument("gateway script: unknown step " + what);
}

std::string op_gateway(const json& job) {
  gateway::Gateway gw(policy_from(job));
  gw.session_ttl_s = job.value("session_ttl_s", 3600.0);
  gw.backend_timeout_s = job.value("backend_timeout_s", 30.0);
  json out = json::array();
  for (const json& it : job.at("script")) out.push_back(gateway_item(gw, it));
  const gateway::GatewayStats s = gw.stats();
  return json{{"results", out}, {"decision_latency_p99_us", s.decision_latency_p99_us}}.dump();
}

// op=gateway_tcp: the gateway on a loopback socket, GPU workers registering and
// heartbeating over the wire (WorkerAgent), then `messages` sent by a client in
// `split`-byte pieces; replies returned in order.
std::string op_gateway_tcp(const json& job) {
  gateway::Gateway gw(policy_from(job));
  std::atomic<bool> stop{false};
  std::atomic<int> port{0};
  int rc = 0;
  std::thread srv([&] { rc = gateway::serve_tcp(gw, job.value("port", 0), stop, &port); });
  for (int i = 0; i < 2000 && port.load() == 0 && rc == 0; ++i) std::this_thread::sleep_for(std::chrono::milliseconds(1));
  json out;
  try {
    if (port.load() == 0) throw std::runtime_error("gateway_tcp: server did not start");
    std::vector<std::unique_ptr<gateway::WorkerAgent>> workers;
    json ids = json::array();
    for (const json& w : job.value("workers", json::array())) {
      workers.push_back(std::make_unique<gateway::WorkerAgent>(
          port.load(), w.at("role").get<std::string>().at(0), w.value("gpu", -1), w.value("address", std::string()),
          job.value("heartbeat_s", 5.0)));
      ids.push_back(workers.back()->id());
    }
    gateway::Connection c(port.load());
    json replies = json::array();
    const std::size_t split = job.value("split", std::size_t{0});
    for (const json& m : job.value("messages", json::array())) replies.push_back(c.call(m.get<std::string>(), split));
    std::this_thread::sleep_for(std::chrono::duration<double>(job.value("hold_s", 0.0)));
    long beats = 0;
    for (const auto& w : workers) beats += w->heartbeats();
    json failed = json::array();
    if (job.value("stop_server_first", false)) {
      // the gateway goes away under live agents: their heartbeat threads must
      // stop cleanly (recorded failure), never terminate the process
      stop.store(true);
      srv.join();
      std::this_thread::sleep_for(std::chrono::duration<double>(job.value("after_stop_s", 0.0)));
      for (const auto& w : workers) failed.push_back({{"failed", w->failed()}, {"error", w->error()}});
    }
    workers.clear();
    out = {{"port", port.load()}, {"worker_ids", ids}, {"replies", replies}, {"heartbeats", beats},
           {"after_stop", failed}};
  } catch (...) {
    stop.store(true);
    if (srv.joinable()) srv.join();
    throw;
  }
  stop.store(true);
  if (srv.joinable()) srv.join();
  return out.dump();
}

// The KV manager alone (ppd::kv::BlockPool): a script of ensure / set_tokens /
// release operations; replies each table after each op (exact block ids).
std::string op_kv_pool_script(const json& job) {
  kv::BlockPool pool(job.at("num_blocks").get<int>(), job.value("block_tokens", 16));
  json out = json::array();
  for (const json& it : job.at("script")) {
    const std::string what = it.at("do").get<std::string>();
    const int conv = it.at("conv").get<int>();
    json r = {{"do", what}, {"conv", conv}};
    try {
      if (what == "ensure") {
        pool.ensure(conv, it.at("tokens").get<long>());
      } else if (what == "set_tokens") {
        pool.set_tokens(conv, it.at("tokens").get<long>());
      } else if (what == "release") {
        pool.release(conv);
      } else {
        throw std::invalid_argument("kv_pool_script: unknown op " + what);
      }
    } catch (const std::runtime_error& e) {
      r["error"] = e.what();
    }
    const kv::BlockTable* t = pool.find(conv);
    r["blocks"] = t ? json(t->blocks) : json::array();
    r["tokens"] = pool.tokens(conv);
    r["free_blocks"] = pool.free_blocks();
    out.push_back(r);
  }
  return out.dump();
}

std::string run(const std::string& text) {
  const json job = json::parse(text);
  const std::string op = job.value("op", std::string("simulate"));
  if (op == "fit_calibration") return fit(job);
  if (op == "build_table") return build_table(job);
  if (op == "sweep") return op_sweep(job);
  if (op == "pareto") return op_pareto(job);
  if (op == "winner") return op_winner(job);
  if (op == "weight_sweep") return op_weight_sweep(job);
  if (op == "plan_default") return op_plan_default();
  if (op == "ingest_trace") return op_ingest_trace(job);
  if (op == "gateway") return op_gateway(job);
  if (op == "gateway_tcp") return op_gateway_tcp(job);
  if (op == "kv_pool_script") return op_kv_pool_script(job);
  auto calib = std::make_shared<const cost::CalibrationTable>(calib_from(job));
  sim::ClusterConfig cfg = sim::ClusterConfig::from_name(job.at("cluster").get<std::string>(), policy_from(job), calib);
  if (job.contains("max_decode_batch")) cfg.max_decode_batch = job["max_decode_batch"].get<int>();
  if (job.contains("request_timeout_s")) cfg.request_timeout_s = job["request_timeout_s"].get<double>();
  if (job.contains("kv_blocks_per_node")) cfg.kv_blocks_per_node = job["kv_blocks_per_node"].get<int>();
  const auto convs = convs_from(job);
  const double qps_replay = job.value("qps_replay", -1.0);
  const std::uint64_t seed = job.value("seed", std::uint64_t{1});
  const double think = job.value("think_time_s", 0.0);
  const auto t0 = std::chrono::steady_clock::now();
  const std::string clock = job.value("clock", std::string("virtual"));
  if (clock == "device" || clock == "realtime") {
    engine::DeviceOptions opt = engine::DeviceOptions::from_json(job.value("device", json::object()).dump());
    opt.realtime = clock == "realtime";
    engine::DeviceRun dr = engine::run_on_device(cfg, convs, qps_replay, seed, think, opt);
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    json out = result_json(dr.sim, job, calib->hash(), wall);
    out["device"] = json::parse(dr.device_json);
    return out.dump();
  }
  const sim::SimResult r = sim::run_simulation(cfg, convs, qps_replay, seed, think);
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return result_json(r, job, calib->hash(), wall).dump();
}

}  // namespace

extern "C" {

int ppd_engine_run_json(const char* job_json, char** out_json) {
  try {
    const std::string s = run(job_json ? job_json : "");
    char* buf = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(buf, s.c_str(), s.size() + 1);
    *out_json = buf;
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

void ppd_engine_free(char* p) { std::free(p); }

struct ppd_gateway {
  gateway::Gateway gw;
  std::atomic<bool> stop{false};
  std::atomic<int> port{0};
  std::thread server;
  explicit ppd_gateway(routing::RoutingPolicy p) : gw(std::move(p)) {}
};

#define PPD_GW_GUARD(body)                          \
  try {                                             \
    body;                                           \
    return 0;                                       \
  } catch (const std::invalid_argument& e) {        \
    g_err = e.what();                               \
    return -1;                                      \
  } catch (const std::exception& e) {               \
    g_err = e.what();                               \
    return -2;                                      \
  }

int ppd_gateway_create(const char* policy_json, ppd_gateway** out) {
  PPD_GW_GUARD({
    if (!out) throw std::invalid_argument("ppd_gateway_create: out is null");
    const json j = json::parse(policy_json && *policy_json ? policy_json : "{}");
    auto* g = new ppd_gateway(policy_from(j));
    g->gw.session_ttl_s = j.value("session_ttl_s", 3600.0);
    g->gw.backend_timeout_s = j.value("backend_timeout_s", 30.0);
    *out = g;
  })
}

int ppd_gateway_handle(ppd_gateway* gw, const char* payload, double now, char** reply) {
  PPD_GW_GUARD({
    if (!gw || !payload || !reply) throw std::invalid_argument("ppd_gateway_handle: null argument");
    const std::string r = gw->gw.handle_message(payload, now);
    char* buf = static_cast<char*>(std::malloc(r.size() + 1));
    std::memcpy(buf, r.c_str(), r.size() + 1);
    *reply = buf;
  })
}

int ppd_gateway_serve(ppd_gateway* gw, int port, int* bound_port) {
  PPD_GW_GUARD({
    if (!gw) throw std::invalid_argument("ppd_gateway_serve: null gateway");
    if (gw->server.joinable()) throw std::invalid_argument("ppd_gateway_serve: already serving");
    if (port < 0 || port > 65535) throw std::invalid_argument("ppd_gateway_serve: bad port");
    gw->stop.store(false);
    gw->port.store(0);
    std::atomic<int> rc{0};
    gw->server = std::thread([gw, port, &rc] {
      if (gateway::serve_tcp(gw->gw, port, gw->stop, &gw->port) < 0) rc.store(-1);
    });
    while (gw->port.load() == 0 && rc.load() == 0) std::this_thread::sleep_for(std::chrono::milliseconds(1));
    if (rc.load() < 0) {
      gw->server.join();
      throw std::runtime_error("ppd_gateway_serve: cannot bind 127.0.0.1:" + std::to_string(port));
    }
    if (bound_port) *bound_port = gw->port.load();
  })
}

int ppd_gateway_stop(ppd_gateway* gw) {
  PPD_GW_GUARD({
    if (!gw) throw std::invalid_argument("ppd_gateway_stop: null gateway");
    gw->stop.store(true);
    if (gw->server.joinable()) gw->server.join();
  })
}

void ppd_gateway_destroy(ppd_gateway* gw) {
  if (!gw) return;
  ppd_gateway_stop(gw);
  delete gw;
}
const char* ppd_engine_last_error(void) { return g_err.c_str(); }

}  // extern "C"
