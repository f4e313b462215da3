// engine.cpp — device-clock execution of the P/D/R cluster (ppd/engine.hpp).
//
// Same request lifecycle, router and session semantics as the virtual clock
// (simulator.cpp, reference simulator.cpp:218-445) with the four analytic
// service times replaced by real work on B200s through the C-ABI:
//   prefill lane + decode loop   -> one fused ppd_step per node iteration
//   kv_transfer_time             -> ppd_kv_copy of the missing tokens
// The engine clock of a node advances by the CUDA-event duration of its own
// step; nodes are independent GPUs (node i -> gpus[i % n]).
#include <cstdlib>
#include <fstream>
#include <algorithm>
#include <cmath>
#include <deque>
#include <map>
#include <memory>
#include <queue>
#include <sstream>
#include <stdexcept>
#include <unordered_map>

#include <json.hpp>

#include "../../include/ppd_b200.h"
#include "ppd/engine.hpp"
#include "ppd/kvcache.hpp"
#include "ppd/util.hpp"

namespace ppd::engine {

using nlohmann::json;

DeviceOptions DeviceOptions::from_json(const std::string& text) {
  const json j = text.empty() ? json::object() : json::parse(text);
  DeviceOptions o;
  o.model.name = j.value("model", std::string("tiny"));
  o.model.n_layers = j.value("n_layers", 0);
  o.weight_seed = j.value("weight_seed", std::uint64_t{1});
  o.token_seed = j.value("token_seed", std::uint64_t{1});
  if (j.contains("gpus")) o.gpus = j["gpus"].get<std::vector<int>>();
  o.kv_blocks_per_node = j.value("kv_blocks_per_node", 0);
  o.prefill_chunk = j.value("prefill_chunk", 2048);
  o.max_step_tokens = j.value("max_step_tokens", 0);
  o.record_steps = j.value("record_steps", false);
  o.record_tokens = j.value("record_tokens", true);
  if (o.gpus.empty()) throw std::invalid_argument("device options: gpus must not be empty");
  if (o.prefill_chunk < 1) throw std::invalid_argument("device options: prefill_chunk must be >= 1");
  return o;
}

namespace {

ppd_model_cfg shape_cfg(const ModelShape& m) {
  ppd_model_cfg c{};
  if (m.name == "tiny") {
    c = {2, 512, 4, 1, 128, 1024, 2048, 1e-5f, 5e5f, 0};
  } else if (m.name == "llama8b") {
    c = {32, 4096, 32, 8, 128, 14336, 128256, 1e-5f, 5e5f, 0};
  } else if (m.name == "qwen32b") {
    c = {64, 5120, 40, 8, 128, 27648, 152064, 1e-6f, 1e6f, 1};
  } else {
    throw std::invalid_argument("unknown model shape: " + m.name);
  }
  if (m.n_layers > 0) c.n_layers = m.n_layers;
  return c;
}

void check(int rc, const char* what) {
  if (rc != PPD_OK) {
    std::string msg = std::string(what) + ": " + ppd_last_error();
    if (rc == PPD_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }
}

enum class Ev { issue, iter_done, transfer_done, timeout };
struct Event {
  double t;
  std::uint64_t seq;
  Ev kind;
  int a, b;
};
struct Later {
  bool operator()(const Event& x, const Event& y) const { return x.t != y.t ? x.t > y.t : x.seq > y.seq; }
};

struct Req {
  int conv, turn;
  double arrival;
  long m, ctx, target;
  long emitted = 0;
  double first = -1, done = -1;
  metrics::Route route = metrics::Route::P_path;
  bool terminal = false, timed_out = false;
  int dnode = -1;
  std::vector<std::int32_t> out;  // generated token ids of this turn
};

struct Job {
  bool full;       // full history recompute (positions 0..) vs append
  int req;
  long begin, end; // positions covered by this job
  long next;       // first position not yet processed
  double enq;
  int key;         // KV table key on the node (conv, or a per-request temp key on P)
};

struct Row {
  int kind;  // 0 decode, 1 flush (KV only), 2 prefill chunk
  int rid, conv;
};

struct Node {
  char role;
  int gpu;
  ppd_dev* dev = nullptr;
  kv::BlockPool pool;
  std::deque<Job> queue;
  bool has_job = false;
  Job job{};
  std::vector<int> running;
  std::deque<int> admit;
  std::vector<int> flush;  // conversations whose last token's KV is pending
  std::unordered_map<int, int> flush_pending;  // conv -> queued or in-flight KV-only rows
  std::vector<std::int32_t> last_out;
  bool busy = false;
  std::vector<Row> rows;
  long chunk = 0;
  bool chunk_final = false;
  double t_prefill = 0, t_decode = 0;
  long steps = 0, decode_rows = 0, prefill_tokens = 0;
  double device_ms = 0;
};

struct Link {
  double egress_free = 0, ingress_free = 0;
};

class DeviceCluster {
 public:
  DeviceCluster(const sim::ClusterConfig& cfg, const std::vector<workload::Conversation>& convs, double qps_replay,
                std::uint64_t seed, double think, const DeviceOptions& opt)
      : cfg_(cfg), convs_(convs), opt_(opt), policy_(cfg.policy), think_(think) {
    cfg_.validate();
    mcfg_ = shape_cfg(opt.model);
    std::uint64_t bb = 0;
    check(ppd_kv_block_bytes(&mcfg_, 16, &bb), "kv block bytes");
    kv_tok_bytes_ = double(bb) / 16.0;
    // KV capacity: every conversation's full history, unless given
    long need_blocks = 64;
    for (const auto& c : convs_) {
      long tot = 0;
      for (const auto& t : c.turns) tot += t.new_input_tokens + t.target_output_tokens;
      need_blocks += (tot + 15) / 16 + 1;
    }
    const int blocks = opt.kv_blocks_per_node > 0 ? opt.kv_blocks_per_node : int(need_blocks);
    max_step_tokens_ = opt.max_step_tokens > 0 ? opt.max_step_tokens
                                               : opt.prefill_chunk + cfg_.max_decode_batch * 2 + 64;
    auto add = [&](char role, int n) {
      for (int i = 0; i < n; ++i) {
        Node nd{role, opt.gpus[nodes_.size() % opt.gpus.size()], nullptr, kv::BlockPool(blocks, 16)};
        nodes_.push_back(std::move(nd));
      }
    };
    add('P', cfg_.p_nodes);
    add('D', cfg_.d_nodes);
    add('R', cfg_.r_nodes);
    for (Node& n : nodes_) {
      check(ppd_dev_open(n.gpu, &mcfg_, max_step_tokens_, cfg_.max_decode_batch * 2 + 8, &n.dev), "dev open");
      check(ppd_load_random_weights(n.dev, opt.weight_seed), "weights");
      check(ppd_kv_pool_init(n.dev, 16, blocks), "kv pool");
    }
    links_.resize(nodes_.size());
    hist_.resize(convs_.size());
    if (qps_replay > 0) {
      Rng arr(seed ^ 0x7265706c6179ull);
      double t = 0;
      for (std::size_t i = 0; i < convs_.size(); ++i) {
        t += arr.exponential(qps_replay);
        push(t, Ev::issue, int(i), 0);
      }
    } else {
      for (std::size_t i = 0; i < convs_.size(); ++i) {
        if (convs_[i].turns.empty()) continue;
        const double t = convs_[i].turns.front().arrival_time;
        if (t < 0) throw std::invalid_argument("conversation lacks a Turn-1 arrival and no qps_replay given");
        push(t, Ev::issue, int(i), 0);
      }
    }
  }

  ~DeviceCluster() {
    for (Node& n : nodes_)
      if (n.dev) ppd_dev_close(n.dev);
  }

  DeviceRun run() {
    while (!q_.empty()) {
      const Event e = q_.top();
      q_.pop();
      now_ = e.t;
      makespan_ = std::max(makespan_, now_);
      switch (e.kind) {
        case Ev::issue: issue(e.a, e.b); break;
        case Ev::iter_done: iter_done(e.a); break;
        case Ev::transfer_done: transfer_done(e.a); break;
        case Ev::timeout: timeout(e.a); break;
      }
    }
    return collect();
  }

 private:
  void push(double t, Ev k, int a, int b = 0) { q_.push(Event{t, seq_++, k, a, b}); }

  double recent_qps() {
    while (!window_.empty() && window_.front() < now_ - 10.0) window_.pop_front();
    return double(window_.size()) / 10.0;
  }
  std::size_t prefill_depth(const Node& n) const { return n.queue.size() + (n.has_job ? 1 : 0); }
  std::size_t decode_depth(const Node& n) const { return n.running.size() + n.admit.size(); }
  int least_loaded(char role, bool by_decode) const {
    int best = -1;
    std::size_t bd = 0;
    for (int i = 0; i < int(nodes_.size()); ++i) {
      if (nodes_[i].role != role) continue;
      const std::size_t d = by_decode ? decode_depth(nodes_[i]) : prefill_depth(nodes_[i]);
      if (best < 0 || d < bd) {
        best = i;
        bd = d;
      }
    }
    return best;
  }

  // ---------------------------------------------------------- lifecycle
  void issue(int conv, int turn) {
    const workload::TurnRequest& tr = convs_[conv].turns[turn];
    const int rid = int(reqs_.size());
    reqs_.push_back(Req{conv, turn, now_, tr.new_input_tokens, tr.cached_context_tokens, tr.target_output_tokens});
    push(now_ + cfg_.request_timeout_s, Ev::timeout, rid);
    if (turn == 0) window_.push_back(now_);
    // the turn's input tokens join the conversation history
    std::vector<std::int32_t>& h = hist_[conv];
    if (long(h.size()) != tr.cached_context_tokens)
      throw std::logic_error("history length != cached context at turn issue");
    for (long p = tr.cached_context_tokens; p < tr.cached_context_tokens + tr.new_input_tokens; ++p)
      h.push_back(std::int32_t(workload::token_id(opt_.token_seed, convs_[conv].first_message_digest, turn, p,
                                                  mcfg_.vocab)));
    const Digest128& key = convs_[conv].first_message_digest;
    if (const auto s = sessions_.find(key); s && s->assigned_pd >= 0 && nodes_[s->assigned_pd].role == 'R' && turn > 0) {
      sessions_.update(key, now_);
      reqs_[rid].route = metrics::Route::R_local;
      reqs_[rid].dnode = s->assigned_pd;
      enqueue(s->assigned_pd, append_job(rid));
      return;
    }
    int pick_p = -1, pick_d = -1;
    auto assign = [&]() {
      const int p = least_loaded('P', false), r = least_loaded('R', false);
      bool replica = p < 0;
      if (p >= 0 && r >= 0) replica = prefill_depth(nodes_[r]) < prefill_depth(nodes_[p]);
      if (replica) {
        pick_p = pick_d = r;
      } else {
        pick_p = p;
        pick_d = least_loaded('D', true);
      }
      return pick_d;
    };
    workload::TurnRequest stamped = tr;
    stamped.arrival_time = now_;
    const routing::RouteDecision dec = routing::decide(stamped, key, recent_qps(), policy_, sessions_, now_, assign);
    if (dec.session_missing) ++session_misses_;
    if (turn > 0) route_log_.push_back(dec.x_used);
    Req& r = reqs_[rid];
    if (dec.target == routing::RouteDecision::Target::D_local) {
      r.route = metrics::Route::D_local;
      r.dnode = sessions_.find(key)->assigned_pd;
      enqueue(r.dnode, append_job(rid));
      return;
    }
    int d = pick_d, p = pick_p;
    if (d < 0) {
      d = sessions_.find(key)->assigned_pd;
      p = least_loaded('P', false);
    }
    r.dnode = d;
    if (nodes_[d].role == 'R') {
      r.route = metrics::Route::R_local;
      enqueue(d, full_job(rid, conv));
      return;
    }
    r.route = metrics::Route::P_path;
    enqueue(p, full_job(rid, -(rid + 1)));  // P recomputes the whole history in a temp table
  }

  Job append_job(int rid) {
    const Req& r = reqs_[rid];
    return Job{false, rid, r.ctx, r.ctx + r.m, r.ctx, now_, r.conv};
  }
  Job full_job(int rid, int key) {
    const Req& r = reqs_[rid];
    return Job{true, rid, 0, r.ctx + r.m, 0, now_, key};
  }

  void enqueue(int node, const Job& j) {
    nodes_[node].queue.push_back(j);
    start_iter(node);
  }

  // ------------------------------------------------------- node iteration
  void start_iter(int ni) {
    Node& n = nodes_[ni];
    if (n.busy) return;
    while (!n.admit.empty() && int(n.running.size()) < cfg_.max_decode_batch) {
      const int rid = n.admit.front();
      n.admit.pop_front();
      if (!reqs_[rid].terminal) n.running.push_back(rid);
    }
    if (n.has_job && reqs_[n.job.req].terminal) drop_job(n);
    while (!n.has_job && !n.queue.empty()) {
      Job j = n.queue.front();
      n.queue.pop_front();
      if (reqs_[j.req].terminal) continue;
      waits_.push_back(now_ - j.enq);
      n.job = j;
      n.has_job = true;
    }
    if (n.running.empty() && n.flush.empty() && !n.has_job) return;

    n.rows.clear();
    std::vector<std::int32_t> q_len, ctx, toks, want;
    std::vector<const std::vector<std::int32_t>*> tables;
    for (int rid : n.running) {
      const Req& r = reqs_[rid];
      const long pos = n.pool.tokens(r.conv);
      const auto& t = n.pool.ensure(r.conv, pos + 1);
      n.rows.push_back({0, rid, r.conv});
      q_len.push_back(1);
      ctx.push_back(std::int32_t(pos));
      toks.push_back(hist_[r.conv][pos]);
      tables.push_back(&t.blocks);
      want.push_back(1);
    }
    const std::vector<int> flushing = std::move(n.flush);
    n.flush.clear();
    for (int conv : flushing) {
      const long pos = n.pool.tokens(conv);
      const auto& t = n.pool.ensure(conv, pos + 1);
      n.rows.push_back({1, -1, conv});
      q_len.push_back(1);
      ctx.push_back(std::int32_t(pos));
      toks.push_back(hist_[conv][pos]);
      tables.push_back(&t.blocks);
      want.push_back(0);
    }
    n.chunk = 0;
    if (n.has_job) {
      Job& j = n.job;
      const Req& r = reqs_[j.req];
      n.chunk = std::min<long>(opt_.prefill_chunk, j.end - j.next);
      n.chunk_final = j.next + n.chunk == j.end;
      const auto& t = n.pool.ensure(j.key, j.next + n.chunk);
      n.rows.push_back({2, j.req, r.conv});
      q_len.push_back(std::int32_t(n.chunk));
      ctx.push_back(std::int32_t(j.next));
      for (long p = j.next; p < j.next + n.chunk; ++p) toks.push_back(hist_[r.conv][p]);
      tables.push_back(&t.blocks);
      want.push_back(n.chunk_final ? 1 : 0);
    }
    std::size_t maxb = 1;
    for (auto* t : tables) maxb = std::max(maxb, t->size());
    std::vector<std::int32_t> bt(tables.size() * maxb, 0);
    for (std::size_t i = 0; i < tables.size(); ++i) std::copy(tables[i]->begin(), tables[i]->end(), bt.begin() + i * maxb);
    ppd_batch b{};
    b.n_seqs = std::int32_t(q_len.size());
    b.q_len = q_len.data();
    b.ctx = ctx.data();
    b.tokens = toks.data();
    b.block_tables = bt.data();
    b.max_blocks = std::int32_t(maxb);
    b.want_token = want.data();
    std::vector<std::int32_t> out(q_len.size(), -1);
    float ms = 0.f;
    check(ppd_step(n.dev, &b, out.data(), &ms), "ppd_step");
    // map outputs (only want rows produce tokens, in row order)
    step_out_.clear();
    for (std::size_t i = 0, k = 0; i < want.size(); ++i) step_out_.push_back(want[i] ? out[k++] : -1);
    // a sampled id outside the vocabulary means non-finite logits: fail here,
    // at the step that produced it, not when it is fed back a step later
    for (std::size_t i = 0; i < want.size(); ++i)
      if (want[i] && (step_out_[i] < 0 || step_out_[i] >= mcfg_.vocab)) {
        if (const char* path = std::getenv("PPD_DUMP_BAD_STEP")) {  // replayable record of the failing step
          std::ofstream f(path);
          f << nlohmann::json{{"node", ni}, {"role", std::string(1, n.role)}, {"q_len", q_len}, {"ctx", ctx},
                              {"tokens", toks}, {"block_tables", bt}, {"max_blocks", maxb}, {"want", want},
                              {"out", step_out_}, {"step", n.steps}}
                   .dump();
        }
        throw std::runtime_error("device step produced token id " + std::to_string(step_out_[i]) + " on node " +
                                 std::to_string(ni) + " (" + std::string(1, n.role) + ") row " + std::to_string(i) +
                                 " of " + std::to_string(want.size()) + ": q_len " + std::to_string(q_len[i]) +
                                 ", ctx " + std::to_string(ctx[i]) + ", step " + std::to_string(n.steps));
      }
    n.steps += 1;
    n.device_ms += ms;
    n.decode_rows += long(n.running.size());
    n.prefill_tokens += n.chunk;
    const double dur = double(ms) * 1e-3;
    if (n.chunk > 0) n.t_prefill += dur;
    if (!n.running.empty()) n.t_decode += dur;
    if (opt_.record_steps) {
      step_log_.push_back({{"node", ni}, {"q_len", q_len}, {"ctx", ctx}, {"tokens", toks}, {"block_tables", bt},
                           {"max_blocks", maxb}, {"want", want}, {"out", step_out_}, {"ms", ms}});
    }
    n.last_out = step_out_;
    n.busy = true;
    push(now_ + dur, Ev::iter_done, ni);
  }

  void drop_job(Node& n) {
    if (n.job.key < 0) n.pool.release(n.job.key);
    n.has_job = false;
  }

  void iter_done(int ni) {
    Node& n = nodes_[ni];
    n.busy = false;
    std::vector<int> still;
    bool job_finished = false;
    for (std::size_t i = 0; i < n.rows.size(); ++i) {
      const Row& row = n.rows[i];
      if (row.kind == 1) {
        n.pool.set_tokens(row.conv, n.pool.tokens(row.conv) + 1);
        if (--n.flush_pending[row.conv] == 0) n.flush_pending.erase(row.conv);
        continue;
      }
      if (row.kind == 2) {
        job_finished = n.chunk_final;
        n.job.next += n.chunk;
        if (!job_finished) continue;
        Req& r = reqs_[row.rid];
        if (r.terminal) {
          drop_job(n);
          continue;
        }
        const std::int32_t first_tok = n.last_out[i];
        hist_[r.conv].push_back(first_tok);
        r.out.push_back(first_tok);
        if (n.role == 'P') {
          ship(ni, row.rid);
        } else {
          n.pool.set_tokens(r.conv, r.ctx + r.m);
          first_token(row.rid, ni);
        }
        n.has_job = false;
        continue;
      }
      // decode row
      Req& r = reqs_[row.rid];
      if (r.terminal) continue;
      n.pool.set_tokens(r.conv, n.pool.tokens(r.conv) + 1);
      const std::int32_t tok = n.last_out[i];
      hist_[r.conv].push_back(tok);
      r.out.push_back(tok);
      if (++r.emitted >= r.target)
        complete(row.rid);
      else
        still.push_back(row.rid);
    }
    // requests admitted during this iteration stay in `admit`; keep the rest running
    n.running = std::move(still);
    start_iter(ni);
  }

  // token 1 exists (sampled from the prefill's last row): the request is live on its decode node
  void first_token(int rid, int dnode) {
    Req& r = reqs_[rid];
    r.emitted = 1;
    r.first = now_;
    if (r.emitted >= r.target) {
      complete(rid);
      return;
    }
    nodes_[dnode].admit.push_back(rid);
  }

  // P finished the full prefill: move the tokens D is missing over the link
  void ship(int pi, int rid) {
    Node& p = nodes_[pi];
    Req& r = reqs_[rid];
    Node& d = nodes_[r.dnode];
    auto fp = d.flush_pending.find(r.conv);
    const long have = d.pool.tokens(r.conv) + (fp == d.flush_pending.end() ? 0 : fp->second);
    const long total = r.ctx + r.m;
    const long need = std::max<long>(1, total - have);
    const long start = total - need;
    const auto& src = p.pool.ensure(p.job.key, total);
    const auto& dst = d.pool.ensure(r.conv, total);
    const std::size_t nb = std::size_t((total + 15) / 16);
    std::vector<std::int32_t> sb(src.blocks.begin(), src.blocks.begin() + nb);
    std::vector<std::int32_t> db(dst.blocks.begin(), dst.blocks.begin() + nb);
    float ms = 0.f;
    check(ppd_kv_copy(p.dev, d.dev, sb.data(), db.data(), std::int32_t(nb), std::int32_t(start), std::int32_t(need), &ms),
          "ppd_kv_copy");
    if (opt_.record_steps)
      step_log_.push_back({{"copy", true}, {"src", pi}, {"dst", r.dnode}, {"src_blocks", sb}, {"dst_blocks", db},
                           {"start", start}, {"n", need}, {"ms", ms}});
    p.pool.release(p.job.key);
    // FIFO on P's egress and D's ingress (NVSwitch: no shared cluster-wide link)
    const double begin = std::max({now_, links_[pi].egress_free, links_[r.dnode].ingress_free});
    const double done = begin + double(ms) * 1e-3;
    links_[pi].egress_free = done;
    links_[r.dnode].ingress_free = done;
    link_.transfers += 1;
    link_.total_bytes += double(need) * kv_tok_bytes_;
    link_.queue_delays.push_back(begin - now_);
    xfer_ms_ += ms;
    xfer_bytes_ += double(need) * kv_tok_bytes_;
    push(done, Ev::transfer_done, rid);
  }

  void transfer_done(int rid) {
    Req& r = reqs_[rid];
    if (r.terminal) return;
    nodes_[r.dnode].pool.set_tokens(r.conv, r.ctx + r.m);
    first_token(rid, r.dnode);
    start_iter(r.dnode);
  }

  void complete(int rid) {
    Req& r = reqs_[rid];
    r.terminal = true;
    r.done = now_;
    Node& d = nodes_[r.dnode];
    // the last sampled token has no KV yet: a KV-only row writes it next iteration
    if (r.turn + 1 < int(convs_[r.conv].turns.size())) {
      d.flush.push_back(r.conv);
      d.flush_pending[r.conv] += 1;
      push(now_ + think_, Ev::issue, r.conv, r.turn + 1);
    }
  }

  void timeout(int rid) {
    Req& r = reqs_[rid];
    if (r.terminal) return;
    r.terminal = true;
    r.timed_out = true;
    if (r.dnode >= 0) std::erase(nodes_[r.dnode].running, rid);
  }

  DeviceRun collect() {
    DeviceRun out;
    sim::SimResult& s = out.sim;
    json tokens = json::object();
    for (const Req& r : reqs_) {
      metrics::RequestRecord rec;
      rec.conv_id = convs_[r.conv].conv_id;
      rec.turn_index = r.turn + 1;
      rec.arrival = r.arrival;
      if (r.first >= 0 && !r.timed_out) rec.first_token = r.first;
      if (!r.timed_out && r.done >= 0) rec.completion = r.done;
      rec.output_tokens_emitted = r.emitted;
      rec.route = r.route;
      rec.status = r.timed_out ? metrics::Status::timed_out : metrics::Status::completed;
      s.records.push_back(std::move(rec));
      if (opt_.record_tokens) tokens[convs_[r.conv].conv_id][std::to_string(r.turn + 1)] = r.out;
    }
    std::stable_sort(s.records.begin(), s.records.end(), [](const metrics::RequestRecord& a, const metrics::RequestRecord& b) {
      if (a.arrival != b.arrival) return a.arrival < b.arrival;
      if (a.conv_id != b.conv_id) return a.conv_id < b.conv_id;
      return a.turn_index < b.turn_index;
    });
    s.link_transfers = link_.transfers;
    s.link_bytes = link_.total_bytes;
    s.link_queue_delays = link_.queue_delays;
    json nodes = json::array();
    for (int i = 0; i < int(nodes_.size()); ++i) {
      const Node& n = nodes_[i];
      s.node_stats.push_back({n.role, n.t_prefill, n.t_decode});
      for (const auto& [key, tab] : n.pool.tables())
        if (key >= 0) s.kv_tables.push_back({i, convs_[key].conv_id, tab.tokens, tab.blocks});
      nodes.push_back({{"role", std::string(1, n.role)}, {"gpu", n.gpu}, {"steps", n.steps},
                       {"decode_rows", n.decode_rows}, {"prefill_tokens", n.prefill_tokens},
                       {"device_ms", n.device_ms}, {"kv_blocks_used", n.pool.used_blocks()}});
    }
    s.makespan = makespan_;
    s.prefill_wait_samples = std::move(waits_);
    s.session_miss_fallbacks = session_misses_;
    s.route_decisions = std::move(route_log_);
    json dj = {{"nodes", nodes},
               {"kv_transfer", {{"transfers", link_.transfers}, {"bytes", xfer_bytes_}, {"device_ms", xfer_ms_},
                                {"gbs", xfer_ms_ > 0 ? xfer_bytes_ / (xfer_ms_ * 1e-3) / 1e9 : 0.0}}},
               {"model", opt_.model.name},
               {"n_layers", mcfg_.n_layers},
               {"kv_bytes_per_token", kv_tok_bytes_},
               {"gpus", opt_.gpus}};
    if (opt_.record_tokens) dj["tokens"] = tokens;
    if (opt_.record_steps) dj["step_log"] = step_log_;
    out.device_json = dj.dump();
    return out;
  }

  sim::ClusterConfig cfg_;
  const std::vector<workload::Conversation>& convs_;
  DeviceOptions opt_;
  ppd_model_cfg mcfg_{};
  double kv_tok_bytes_ = 0;
  int max_step_tokens_ = 0;
  routing::RoutingPolicy policy_;
  routing::SessionTable sessions_;
  std::vector<Node> nodes_;
  std::vector<Link> links_;
  std::vector<Req> reqs_;
  std::vector<std::vector<std::int32_t>> hist_;
  std::priority_queue<Event, std::vector<Event>, Later> q_;
  std::deque<double> window_;
  std::vector<double> waits_;
  std::vector<int> route_log_;
  std::vector<std::int32_t> step_out_;
  json step_log_ = json::array();
  cost::LinkState link_;
  double xfer_ms_ = 0, xfer_bytes_ = 0;
  std::uint64_t seq_ = 0;
  double now_ = 0, makespan_ = 0, think_;
  long session_misses_ = 0;
};

}  // namespace

DeviceRun run_on_device(const sim::ClusterConfig& cfg, const std::vector<workload::Conversation>& convs,
                        double qps_replay, std::uint64_t seed, double think_time_s, const DeviceOptions& opt) {
  DeviceCluster c(cfg, convs, qps_replay, seed, think_time_s, opt);
  return c.run();
}

routing::BenchmarkRunner device_benchmark_runner(const std::string& cluster, const DeviceOptions& opt,
                                                 std::shared_ptr<const cost::CalibrationTable> calib,
                                                 std::vector<std::uint64_t> seeds) {
  return [=](const routing::GridSpec& g, int x) -> std::optional<std::pair<double, double>> {
    try {
      double ttft = 0, tpot = 0;
      int n = 0;
      for (std::uint64_t s : seeds) {
        auto convs = workload::generate_conversations(g.spec, s);
        auto cfg = sim::ClusterConfig::from_name(cluster, routing::RoutingPolicy::static_policy(double(x)), calib);
        DeviceRun r = run_on_device(cfg, convs, -1, s, g.spec.think_time_s, opt);
        auto agg = metrics::aggregate(r.sim.records, std::max(g.spec.duration_s, r.sim.makespan));
        if (!agg.ttft_t2_mean || !agg.tpot_mean) return std::nullopt;
        ttft += *agg.ttft_t2_mean;
        tpot += *agg.tpot_mean;
        ++n;
      }
      if (n == 0) return std::nullopt;
      return std::make_pair(ttft / n, tpot / n);
    } catch (const std::exception&) {
      return std::nullopt;
    }
  };
}

}  // namespace ppd::engine
