// engine.cpp — device-clock and real-time execution of the P/D/R cluster
// (ppd/engine.hpp).
//
// Same request lifecycle, router and session semantics as the virtual clock
// (simulator.cpp, reference simulator.cpp:218-445) with the four analytic
// service times replaced by real work on B200s through the C-ABI:
//   prefill lane + decode loop   -> one fused ppd_step per node iteration
//   kv_transfer_time             -> ppd_kv_copy of the missing tokens
//
// Two clocks drive the same handlers:
//  * device (deterministic): one host thread runs every step synchronously and
//    a node's clock advances by the CUDA-event duration of its own step, so
//    nodes behave as independent GPUs even when they share one.
//  * realtime: the cluster runs in wall-clock time. Each node has a worker
//    thread that submits its steps (ppd_step_submit / ppd_step_wait), every
//    P->D hop is an asynchronous ppd_kv_copy_submit on the destination's
//    transfer stream that overlaps the destination's decode steps, and a
//    per-destination waiter retires the copies; all scheduling state is owned
//    by the event-loop thread, which the workers feed through a mailbox.
//
// KV lifecycle: a conversation's block table on its decode node is released
// when its last turn completes or a turn times out (its later turns are never
// issued, reference simulator.cpp:436-445); P-side temporary tables when their
// hop has landed. Admission control keeps decode rows able to grow: a prefill
// job starts only when its remaining blocks fit beside one block of headroom
// per decode request, hops wait for room on the destination, and a row that
// cannot get a block sits out the iteration instead of aborting the run.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <deque>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <queue>
#include <sstream>
#include <stdexcept>
#include <thread>
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
  o.p_prefill_chunk = j.value("p_prefill_chunk", 8192);
  o.max_step_tokens = j.value("max_step_tokens", 0);
  o.record_steps = j.value("record_steps", false);
  o.record_tokens = j.value("record_tokens", true);
  o.realtime = j.value("realtime", false);
  if (o.gpus.empty()) throw std::invalid_argument("device options: gpus must not be empty");
  if (o.prefill_chunk < 1 || o.p_prefill_chunk < 1)
    throw std::invalid_argument("device options: prefill_chunk and p_prefill_chunk must be >= 1");
  if (o.kv_blocks_per_node < 0) throw std::invalid_argument("device options: kv_blocks_per_node must be >= 0");
  return o;
}

namespace {

ppd_model_cfg model_cfg(const ModelShape& m) {
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

struct DevCloser {
  void operator()(ppd_dev* d) const {
    if (d) ppd_dev_close(d);
  }
};
using DevPtr = std::unique_ptr<ppd_dev, DevCloser>;

// kick: a node picks its next iteration only after every event of the current
// instant (see iter_done)
enum class Ev { issue, iter_done, transfer_done, timeout, kick };
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
  int pnode = -1;            // P node holding the request's temporary table until its hop landed
  bool copy_inflight = false;
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
  long pos;  // first position the row writes
};

// ------------------------------------------------------------ realtime plumbing
using Clock = std::chrono::steady_clock;

struct Done {
  Ev kind;
  int a;
  double t;
  float ms;
  std::vector<std::int32_t> out;
  std::string err;
};

class Mailbox {
 public:
  void post(Done d) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      q_.push_back(std::move(d));
    }
    cv_.notify_one();
  }
  // waits until something is posted or `until` passes; returns what is queued
  std::deque<Done> take(std::optional<Clock::time_point> until) {
    std::unique_lock<std::mutex> lk(mu_);
    if (q_.empty()) {
      if (until)
        cv_.wait_until(lk, *until, [&] { return !q_.empty(); });
      else
        cv_.wait(lk, [&] { return !q_.empty(); });
    }
    std::deque<Done> out;
    out.swap(q_);
    return out;
  }

 private:
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Done> q_;
};

struct StepJob {
  std::vector<std::int32_t> q_len, ctx, toks, bt, want;
  int maxb = 1;
};

// One thread per node: submits the node's steps and reports their completion.
class StepWorker {
 public:
  StepWorker(ppd_dev* dev, int node, Mailbox* mb, Clock::time_point t0)
      : dev_(dev), node_(node), mb_(mb), t0_(t0), th_([this] { loop(); }) {}
  ~StepWorker() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_one();
    th_.join();
  }
  void submit(StepJob j) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = std::move(j);
    }
    cv_.notify_one();
  }

 private:
  void loop() {
    for (;;) {
      StepJob j;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || job_.has_value(); });
        if (stop_) return;
        j = std::move(*job_);
        job_.reset();
      }
      ppd_batch b{};
      b.n_seqs = std::int32_t(j.q_len.size());
      b.q_len = j.q_len.data();
      b.ctx = j.ctx.data();
      b.tokens = j.toks.data();
      b.block_tables = j.bt.data();
      b.max_blocks = j.maxb;
      b.want_token = j.want.data();
      std::vector<std::int32_t> out(j.q_len.size(), -1);
      float ms = 0.f;
      Done d{Ev::iter_done, node_, 0, 0, {}, {}};
      int rc = ppd_step_submit(dev_, &b);
      if (rc == PPD_OK) rc = ppd_step_wait(dev_, out.data(), &ms);
      d.t = std::chrono::duration<double>(Clock::now() - t0_).count();
      if (rc != PPD_OK) d.err = std::string("ppd_step: ") + ppd_last_error();
      d.ms = ms;
      d.out = std::move(out);
      mb_->post(std::move(d));
    }
  }
  ppd_dev* dev_;
  int node_;
  Mailbox* mb_;
  Clock::time_point t0_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::optional<StepJob> job_;
  bool stop_ = false;
  std::thread th_;  // last: starts after the members it uses
};

// One thread per destination node: retires its KV hops in submission order.
class CopyWaiter {
 public:
  CopyWaiter(ppd_dev* dst, Mailbox* mb, Clock::time_point t0) : dst_(dst), mb_(mb), t0_(t0), th_([this] { loop(); }) {}
  ~CopyWaiter() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_one();
    th_.join();
  }
  void add(std::uint64_t ticket, int rid) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      q_.push_back({ticket, rid});
    }
    cv_.notify_one();
  }

 private:
  void loop() {
    for (;;) {
      std::pair<std::uint64_t, int> it;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return !q_.empty() || stop_; });
        if (q_.empty()) return;  // stop requested and drained
        it = q_.front();
        q_.pop_front();
      }
      float ms = 0.f;
      Done d{Ev::transfer_done, it.second, 0, 0, {}, {}};
      if (ppd_kv_copy_wait(dst_, it.first, &ms) != PPD_OK) d.err = std::string("ppd_kv_copy_wait: ") + ppd_last_error();
      d.t = std::chrono::duration<double>(Clock::now() - t0_).count();
      d.ms = ms;
      mb_->post(std::move(d));
    }
  }
  ppd_dev* dst_;
  Mailbox* mb_;
  Clock::time_point t0_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::pair<std::uint64_t, int>> q_;
  bool stop_ = false;
  std::thread th_;
};

struct Node {
  char role;
  int gpu;
  DevPtr dev;  // declared before the threads: they are joined first
  kv::BlockPool pool;
  std::deque<Job> queue;
  bool has_job = false;
  Job job{};
  std::vector<int> running;
  std::deque<int> admit;
  std::vector<int> flush;                      // conversations whose last token's KV is pending
  std::unordered_map<int, int> flush_pending;  // conv -> queued or in-flight KV-only rows
  std::vector<int> release_pending;            // conv tables to return once no step / hop uses them
  std::unordered_map<int, int> copies_in;      // conv -> hops in flight into this node
  std::deque<int> ship_wait;                   // P-path requests waiting for room in this pool
  std::unordered_map<int, double> last_use;    // conv -> last step / hop that touched its table
  std::vector<std::int32_t> last_out;
  bool busy = false;
  std::vector<Row> rows;
  long chunk = 0;
  bool chunk_final = false;
  double t_prefill = 0, t_decode = 0;
  long steps = 0, decode_rows = 0, prefill_tokens = 0, stalled_rows = 0, admission_waits = 0, evictions = 0;
  long peak_blocks = 0;
  double device_ms = 0;
  std::size_t log_idx = 0;  // step-log entry of the in-flight step
  std::unique_ptr<StepWorker> worker;
  std::unique_ptr<CopyWaiter> copier;
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
    mcfg_ = model_cfg(opt.model);
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
    // P nodes run prefill only (no decode rows to protect): larger chunks
    p_step_tokens_ = opt.max_step_tokens > 0 ? opt.max_step_tokens : std::max(opt.p_prefill_chunk, 64);
    auto add = [&](char role, int n) {
      for (int i = 0; i < n; ++i) {
        Node nd;
        nd.role = role;
        nd.gpu = opt.gpus[nodes_.size() % opt.gpus.size()];
        nd.pool = kv::BlockPool(blocks, 16);
        nodes_.push_back(std::move(nd));
      }
    };
    add('P', cfg_.p_nodes);
    add('D', cfg_.d_nodes);
    add('R', cfg_.r_nodes);
    // a failure part-way releases every device already opened (RAII handles)
    for (Node& n : nodes_) {
      ppd_dev* d = nullptr;
      // P nodes run one prefill job per step (serial lane): few sequences
      const int seqs = cfg_.max_decode_batch * 2 + 8;
      check(ppd_dev_open(n.gpu, &mcfg_, n.role == 'P' ? p_step_tokens_ : max_step_tokens_,
                         n.role == 'P' ? std::min(seqs, p_step_tokens_) : std::min(seqs, max_step_tokens_), &d),
            "dev open");
      n.dev.reset(d);
      check(ppd_load_random_weights(d, opt.weight_seed), "weights");
      check(ppd_kv_pool_init(d, 16, blocks), "kv pool");
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
    for (Node& n : nodes_) {
      n.worker.reset();
      n.copier.reset();
    }
  }

  DeviceRun run() {
    if (opt_.realtime)
      run_realtime();
    else
      run_device_clock();
    return collect();
  }

 private:
  // ------------------------------------------------------------ event loops
  void dispatch(const Event& e) {
    switch (e.kind) {
      case Ev::issue: issue(e.a, e.b); break;
      case Ev::iter_done: iter_done(e.a); break;
      case Ev::transfer_done: transfer_done(e.a); break;
      case Ev::timeout: timeout(e.a); break;
      case Ev::kick: start_iter(e.a); break;
    }
  }

  void run_device_clock() {
    while (!q_.empty()) {
      const Event e = q_.top();
      q_.pop();
      now_ = e.t;
      makespan_ = std::max(makespan_, now_);
      dispatch(e);
    }
  }

  void run_realtime() {
    t0_ = Clock::now();
    for (std::size_t i = 0; i < nodes_.size(); ++i) {
      nodes_[i].worker = std::make_unique<StepWorker>(nodes_[i].dev.get(), int(i), &mb_, t0_);
      if (nodes_[i].role != 'P') nodes_[i].copier = std::make_unique<CopyWaiter>(nodes_[i].dev.get(), &mb_, t0_);
    }
    auto wall = [&] { return std::chrono::duration<double>(Clock::now() - t0_).count(); };
    for (;;) {
      // timers that are due (timeouts of finished requests are dropped unwaited)
      while (!q_.empty()) {
        const Event e = q_.top();
        if (e.kind == Ev::timeout && reqs_[e.a].terminal) {
          q_.pop();
          continue;
        }
        if (e.t > wall()) break;
        q_.pop();
        now_ = std::max(now_, wall());
        makespan_ = std::max(makespan_, now_);
        dispatch(e);
      }
      if (q_.empty() && inflight_steps_ == 0 && inflight_copies_ == 0) break;
      std::optional<Clock::time_point> until;
      if (!q_.empty())
        until = t0_ + std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(q_.top().t));
      for (Done& d : mb_.take(until)) {
        if (!d.err.empty()) throw std::runtime_error(d.err);
        now_ = std::max(now_, d.t);
        makespan_ = std::max(makespan_, now_);
        if (d.kind == Ev::iter_done) {
          --inflight_steps_;
          Node& n = nodes_[d.a];
          n.last_out = std::move(d.out);
          finish_step(d.a, d.ms);
          iter_done(d.a);
        } else {
          --inflight_copies_;
          xfer_ms_ += d.ms;
          hop_ms_.push_back(d.ms);
          transfer_done(d.a);
        }
      }
    }
  }

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
      enqueue(s->assigned_pd, append_job(rid, s->assigned_pd));
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
      enqueue(r.dnode, append_job(rid, r.dnode));
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
    r.pnode = p;
    enqueue(p, full_job(rid, -(rid + 1)));  // P recomputes the whole history in a temp table
  }

  // an append over the node's cached context; a cache evicted under memory
  // pressure is recomputed from position 0 on the node instead
  Job append_job(int rid, int node) {
    const Req& r = reqs_[rid];
    // (a pending completion flush still counts as cached: it runs before the append)
    if (r.ctx > 0 && nodes_[node].pool.find(r.conv) == nullptr) return Job{true, rid, 0, r.ctx + r.m, 0, now_, r.conv};
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
    try_release(ni);
    drain_ship_wait(ni);
    while (!n.admit.empty() && int(n.running.size()) < cfg_.max_decode_batch) {
      const int rid = n.admit.front();
      n.admit.pop_front();
      if (!reqs_[rid].terminal) n.running.push_back(rid);
    }
    if (n.has_job && reqs_[n.job.req].terminal) drop_job(n);
    // headroom kept for the decode rows: one block each (they grow by one token per iteration)
    const long reserve = long(n.running.size() + n.admit.size() + n.flush.size());
    while (!n.has_job && !n.queue.empty()) {
      Job j = n.queue.front();
      if (reqs_[j.req].terminal) {
        n.queue.pop_front();
        continue;
      }
      // admission: the job's remaining blocks must fit beside the decode headroom
      const int need = n.pool.blocks_needed(j.key, j.end) + int(reserve);
      if (need > n.pool.free_blocks() && !evict_for(ni, need, j.key)) {
        ++n.admission_waits;
        break;
      }
      n.queue.pop_front();
      waits_.push_back(now_ - j.enq);
      n.job = j;
      n.has_job = true;
    }

    n.rows.clear();
    std::vector<std::int32_t> q_len, ctx, toks, want;
    std::vector<const std::vector<std::int32_t>*> tables;
    std::vector<int> stalled;
    for (int rid : n.running) {
      const Req& r = reqs_[rid];
      const long pos = n.pool.tokens(r.conv);
      const int need = n.pool.blocks_needed(r.conv, pos + 1);
      if (need > n.pool.free_blocks() && !evict_for(ni, need, r.conv)) {  // sits this iteration out
        stalled.push_back(rid);
        ++n.stalled_rows;
        continue;
      }
      n.last_use[r.conv] = now_;
      const auto& t = n.pool.ensure(r.conv, pos + 1);
      n.rows.push_back({0, rid, r.conv, pos});
      q_len.push_back(1);
      ctx.push_back(std::int32_t(pos));
      toks.push_back(hist_[r.conv][pos]);
      tables.push_back(&t.blocks);
      want.push_back(1);
    }
    std::vector<int> flushing = std::move(n.flush);
    n.flush.clear();
    for (int conv : flushing) {
      const long pos = n.pool.tokens(conv);
      if (n.pool.blocks_needed(conv, pos + 1) > n.pool.free_blocks()) {
        n.flush.push_back(conv);  // retried next iteration
        continue;
      }
      const auto& t = n.pool.ensure(conv, pos + 1);
      n.rows.push_back({1, -1, conv, pos});
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
      const long chunk_cap = n.role == 'P' ? std::min<long>(opt_.p_prefill_chunk, p_step_tokens_) : opt_.prefill_chunk;
      const long c = std::min<long>(chunk_cap, j.end - j.next);
      if (n.pool.blocks_needed(j.key, j.next + c) <= n.pool.free_blocks()) {
        n.chunk = c;
        n.chunk_final = j.next + n.chunk == j.end;
        n.last_use[j.key] = now_;
        const auto& t = n.pool.ensure(j.key, j.next + n.chunk);
        n.rows.push_back({2, j.req, r.conv, j.next});
        q_len.push_back(std::int32_t(n.chunk));
        ctx.push_back(std::int32_t(j.next));
        for (long p = j.next; p < j.next + n.chunk; ++p) toks.push_back(hist_[r.conv][p]);
        tables.push_back(&t.blocks);
        want.push_back(n.chunk_final ? 1 : 0);
      }
    }
    if (n.rows.empty()) return;  // idle (or every row waits for blocks: a release restarts the node)
    n.peak_blocks = std::max<long>(n.peak_blocks, n.pool.used_blocks());
    std::size_t maxb = 1;
    for (auto* t : tables) maxb = std::max(maxb, t->size());
    std::vector<std::int32_t> bt(tables.size() * maxb, 0);
    for (std::size_t i = 0; i < tables.size(); ++i) std::copy(tables[i]->begin(), tables[i]->end(), bt.begin() + i * maxb);
    n.busy = true;
    if (opt_.record_steps) {
      n.log_idx = step_log_.size();
      step_log_.push_back({{"node", ni}, {"q_len", q_len}, {"ctx", ctx}, {"tokens", toks}, {"block_tables", bt},
                           {"max_blocks", maxb}, {"want", want}, {"t_start", now_}});
      if (n.chunk > 0) {  // the prefill chunk's request: when it arrived, which turn
        const Req& r = reqs_[n.job.req];
        step_log_.back()["chunk_req"] = {{"arrival", r.arrival}, {"turn", r.turn}, {"final", n.chunk_final}};
      }
    }
    if (opt_.realtime) {
      ++inflight_steps_;
      n.worker->submit(StepJob{q_len, ctx, toks, std::move(bt), std::move(want), int(maxb)});
      return;
    }
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
    check(ppd_step(n.dev.get(), &b, out.data(), &ms), "ppd_step");
    n.last_out = std::move(out);
    finish_step(ni, ms);
    push(now_ + double(ms) * 1e-3, Ev::iter_done, ni);
  }

  // bookkeeping of a finished step: outputs to row order, sanity, stats
  void finish_step(int ni, float ms) {
    Node& n = nodes_[ni];
    step_out_.clear();
    for (std::size_t i = 0, k = 0; i < n.rows.size(); ++i) {
      const bool want = n.rows[i].kind == 0 || (n.rows[i].kind == 2 && n.chunk_final);
      step_out_.push_back(want ? n.last_out[k++] : -1);
    }
    // a sampled id outside the vocabulary means non-finite logits: fail here,
    // at the step that produced it, not when it is fed back a step later
    for (std::size_t i = 0; i < n.rows.size(); ++i) {
      const bool want = n.rows[i].kind == 0 || (n.rows[i].kind == 2 && n.chunk_final);
      if (want && (step_out_[i] < 0 || step_out_[i] >= mcfg_.vocab))
        throw std::runtime_error("device step produced token id " + std::to_string(step_out_[i]) + " on node " +
                                 std::to_string(ni) + " (" + std::string(1, n.role) + ") row " + std::to_string(i) +
                                 " of " + std::to_string(n.rows.size()) + ", step " + std::to_string(n.steps));
    }
    n.steps += 1;
    n.device_ms += ms;
    long dec = 0;
    for (const Row& r : n.rows) dec += r.kind == 0;
    n.decode_rows += dec;
    n.prefill_tokens += n.chunk;
    const double dur = double(ms) * 1e-3;
    if (n.chunk > 0) n.t_prefill += dur;
    if (dec > 0) n.t_decode += dur;
    if (opt_.record_steps) {
      step_log_[n.log_idx]["out"] = step_out_;
      step_log_[n.log_idx]["ms"] = ms;
    }
    n.last_out = step_out_;
  }

  void drop_job(Node& n) {
    if (n.job.key < 0) n.pool.release(n.job.key);
    n.has_job = false;
  }

  void iter_done(int ni) {
    Node& n = nodes_[ni];
    n.busy = false;
    std::vector<int> still;
    for (std::size_t i = 0; i < n.rows.size(); ++i) {
      const Row& row = n.rows[i];
      if (row.kind == 1) {
        // a hop that landed while this flush ran may already cover more tokens
        n.pool.set_tokens(row.conv, std::max(n.pool.tokens(row.conv), row.pos + 1));
        if (--n.flush_pending[row.conv] == 0) n.flush_pending.erase(row.conv);
        continue;
      }
      if (row.kind == 2) {
        const bool job_finished = n.chunk_final;
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
        n.has_job = false;
        if (n.role == 'P') {
          ship(ni, row.rid);
        } else {
          n.pool.set_tokens(r.conv, r.ctx + r.m);
          first_token(row.rid, ni);
        }
        continue;
      }
      // decode row
      Req& r = reqs_[row.rid];
      if (r.terminal) continue;
      n.pool.set_tokens(r.conv, std::max(n.pool.tokens(r.conv), row.pos + 1));
      const std::int32_t tok = n.last_out[i];
      hist_[r.conv].push_back(tok);
      r.out.push_back(tok);
      if (++r.emitted >= r.target)
        complete(row.rid);
      else
        still.push_back(row.rid);
    }
    // rows that sat out (no free block) stay running; requests admitted during
    // this iteration stay in `admit`
    for (int rid : n.running)
      if (!reqs_[rid].terminal && std::find_if(n.rows.begin(), n.rows.end(), [&](const Row& r) {
                                    return r.kind == 0 && r.rid == rid;
                                  }) == n.rows.end())
        still.push_back(rid);
    n.running = std::move(still);
    // The next iteration is assembled after every event of this instant has
    // been handled: the next turn of a conversation that completed in this
    // step (issued at now + think, think 0 in the configs' traces) joins it
    // instead of waiting a whole step behind it. With the reference's separate
    // prefill lane (simulator.cpp:319-339) such an append starts at once; in
    // the fused step it can only start at an iteration boundary, this one.
    push(now_, Ev::kick, ni);
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
    Req& r = reqs_[rid];
    Node& d = nodes_[r.dnode];
    const long total = r.ctx + r.m;
    const int need = d.pool.blocks_needed(r.conv, total);
    if (!d.ship_wait.empty() || (need > d.pool.free_blocks() && !evict_for(r.dnode, need, r.conv))) {
      d.ship_wait.push_back(rid);  // P keeps its temp table until D has room
      return;
    }
    d.last_use[r.conv] = now_;
    do_ship(pi, rid);
  }

  void do_ship(int pi, int rid) {
    Node& p = nodes_[pi];
    Req& r = reqs_[rid];
    Node& d = nodes_[r.dnode];
    auto fp = d.flush_pending.find(r.conv);
    const long have = d.pool.tokens(r.conv) + (fp == d.flush_pending.end() ? 0 : fp->second);
    const long total = r.ctx + r.m;
    const long need = std::max<long>(1, total - have);
    const long start = total - need;
    const int key = -(rid + 1);
    const auto& src = p.pool.ensure(key, total);
    const auto& dst = d.pool.ensure(r.conv, total);
    const std::size_t nb = std::size_t((total + 15) / 16);
    std::vector<std::int32_t> sb(src.blocks.begin(), src.blocks.begin() + nb);
    std::vector<std::int32_t> db(dst.blocks.begin(), dst.blocks.begin() + nb);
    d.peak_blocks = std::max<long>(d.peak_blocks, d.pool.used_blocks());
    link_.transfers += 1;
    link_.total_bytes += double(need) * kv_tok_bytes_;
    xfer_bytes_ += double(need) * kv_tok_bytes_;
    if (opt_.record_steps)
      step_log_.push_back({{"copy", true}, {"src", pi}, {"dst", r.dnode}, {"src_blocks", sb}, {"dst_blocks", db},
                           {"start", start}, {"n", need}});
    r.copy_inflight = true;
    d.copies_in[r.conv] += 1;
    if (opt_.realtime) {
      std::uint64_t ticket = 0;
      check(ppd_kv_copy_submit(p.dev.get(), d.dev.get(), sb.data(), db.data(), std::int32_t(nb), std::int32_t(start),
                               std::int32_t(need), &ticket),
            "ppd_kv_copy_submit");
      ++inflight_copies_;
      link_.queue_delays.push_back(0.0);
      d.copier->add(ticket, rid);
      return;
    }
    float ms = 0.f;
    check(ppd_kv_copy(p.dev.get(), d.dev.get(), sb.data(), db.data(), std::int32_t(nb), std::int32_t(start),
                      std::int32_t(need), &ms),
          "ppd_kv_copy");
    if (opt_.record_steps) step_log_.back()["ms"] = ms;
    // FIFO on P's egress and D's ingress (NVSwitch: no shared cluster-wide link)
    const double begin = std::max({now_, links_[pi].egress_free, links_[r.dnode].ingress_free});
    const double done = begin + double(ms) * 1e-3;
    links_[pi].egress_free = done;
    links_[r.dnode].ingress_free = done;
    link_.queue_delays.push_back(begin - now_);
    xfer_ms_ += ms;
    hop_ms_.push_back(ms);
    push(done, Ev::transfer_done, rid);
  }

  void drain_ship_wait(int di) {
    Node& d = nodes_[di];
    while (!d.ship_wait.empty()) {
      const int rid = d.ship_wait.front();
      Req& r = reqs_[rid];
      if (r.terminal) {  // timed out while waiting: its P temp table goes back
        d.ship_wait.pop_front();
        release_temp(rid);
        continue;
      }
      const int need = d.pool.blocks_needed(r.conv, r.ctx + r.m);
      if (need > d.pool.free_blocks() && !evict_for(di, need, r.conv)) break;
      d.ship_wait.pop_front();
      d.last_use[r.conv] = now_;
      do_ship(r.pnode, rid);
    }
  }

  void release_temp(int rid) {
    Req& r = reqs_[rid];
    if (r.pnode < 0) return;
    nodes_[r.pnode].pool.release(-(rid + 1));
    const int p = r.pnode;
    r.pnode = -1;
    start_iter(p);  // blocks came back: a waiting job may be admitted
  }

  void transfer_done(int rid) {
    Req& r = reqs_[rid];
    Node& d = nodes_[r.dnode];
    r.copy_inflight = false;
    if (--d.copies_in[r.conv] == 0) d.copies_in.erase(r.conv);
    release_temp(rid);  // the hop read P's temporary table: only now can it be reused
    if (r.terminal) {
      try_release(r.dnode);
      start_iter(r.dnode);
      return;
    }
    d.pool.set_tokens(r.conv, std::max(d.pool.tokens(r.conv), r.ctx + r.m));
    first_token(rid, r.dnode);
    start_iter(r.dnode);
  }

  void complete(int rid) {
    Req& r = reqs_[rid];
    r.terminal = true;
    r.done = now_;
    Node& d = nodes_[r.dnode];
    // coverage invariant: every position but the last sampled token's holds KV
    if (d.pool.tokens(r.conv) != r.ctx + r.m + r.target - 1) ++coverage_errors_;
    if (r.turn + 1 < int(convs_[r.conv].turns.size())) {
      // the last sampled token has no KV yet: a KV-only row writes it next iteration
      d.flush.push_back(r.conv);
      d.flush_pending[r.conv] += 1;
      push(now_ + think_, Ev::issue, r.conv, r.turn + 1);
    } else {
      release_conv(r.dnode, r.conv, false);  // conversation over: its cache is dead
    }
  }

  void timeout(int rid) {
    Req& r = reqs_[rid];
    if (r.terminal) return;
    r.terminal = true;
    r.timed_out = true;
    if (r.dnode >= 0) {
      std::erase(nodes_[r.dnode].running, rid);
      // no later turn of this conversation is ever issued (simulator.cpp:436-445)
      release_conv(r.dnode, r.conv, true);
    }
  }

  // Memory pressure: frees idle conversation caches on node ni (least
  // recently used first) until `need` blocks are free. Idle = no request of
  // the conversation runs, waits for admission or a flush, or receives a hop
  // here; `keep` is the conversation the blocks are for. A queued append of an
  // evicted conversation becomes a full recompute on the node; a later P-path
  // hop ships the whole history (have = 0). Not modelled by the reference
  // (its prefix_cache has no capacity). Only while the node is
  // not stepping: the in-flight step may read any resident table.
  bool evict_for(int ni, int need, int keep) {
    Node& n = nodes_[ni];
    if (n.busy) return false;
    while (n.pool.free_blocks() < need) {
      std::unordered_map<int, bool> busy_conv;
      busy_conv[keep] = true;
      for (int rid : n.running) busy_conv[reqs_[rid].conv] = true;
      for (int rid : n.admit) busy_conv[reqs_[rid].conv] = true;
      if (n.has_job) busy_conv[n.job.key] = true;
      for (int c : n.flush) busy_conv[c] = true;
      for (const auto& [c, k] : n.flush_pending) busy_conv[c] = true;
      for (const auto& [c, k] : n.copies_in) busy_conv[c] = true;
      for (int rid : n.ship_wait) busy_conv[reqs_[rid].conv] = true;
      int victim = -1;
      double oldest = 0;
      for (const auto& [key, tab] : n.pool.tables()) {
        if (key < 0 || busy_conv.count(key) || tab.blocks.empty()) continue;
        auto it = n.last_use.find(key);
        const double t = it == n.last_use.end() ? -1.0 : it->second;
        if (victim < 0 || t < oldest) {
          victim = key;
          oldest = t;
        }
      }
      if (victim < 0) return false;
      if (const kv::BlockTable* t = n.pool.find(victim)) evicted_tokens_ += t->tokens;
      n.pool.release(victim);
      n.last_use.erase(victim);
      ++n.evictions;
      for (Job& j : n.queue)
        if (j.key == victim && !j.full) {
          j.full = true;
          j.begin = j.next = 0;
        }
    }
    return true;
  }

  // a conversation's table on node ni goes back to the pool once no step and
  // no incoming hop touches it. kick: restart the node if idle (only from
  // top-level events; inside iter_done / transfer_done the caller restarts it)
  void release_conv(int ni, int conv, bool kick) {
    Node& n = nodes_[ni];
    n.release_pending.push_back(conv);
    try_release(ni);
    if (kick && !n.busy) start_iter(ni);
  }

  void try_release(int ni) {
    Node& n = nodes_[ni];
    if (n.busy || n.release_pending.empty()) return;
    std::vector<int> keep;
    for (int conv : n.release_pending) {
      if (n.copies_in.count(conv)) {
        keep.push_back(conv);
        continue;
      }
      std::erase(n.flush, conv);
      n.flush_pending.erase(conv);
      if (const kv::BlockTable* t = n.pool.find(conv)) released_tokens_ += t->tokens;
      n.pool.release(conv);
      ++released_tables_;
    }
    n.release_pending = std::move(keep);
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
    long blocks_in_use = 0;
    for (int i = 0; i < int(nodes_.size()); ++i) {
      const Node& n = nodes_[i];
      s.node_stats.push_back({n.role, n.t_prefill, n.t_decode});
      for (const auto& [key, tab] : n.pool.tables())
        if (key >= 0) s.kv_tables.push_back({i, convs_[key].conv_id, tab.tokens, tab.blocks});
      blocks_in_use += n.pool.used_blocks();
      std::uint64_t wbytes = 0;
      std::int32_t wshare = 0;
      ppd_weights_info(n.dev.get(), &wbytes, &wshare);
      nodes.push_back({{"role", std::string(1, n.role)}, {"gpu", n.gpu}, {"steps", n.steps},
                       {"decode_rows", n.decode_rows}, {"prefill_tokens", n.prefill_tokens},
                       {"device_ms", n.device_ms}, {"kv_blocks_used", n.pool.used_blocks()},
                       {"kv_blocks_peak", n.peak_blocks}, {"kv_blocks_total", n.pool.num_blocks()},
                       {"stalled_rows", n.stalled_rows}, {"admission_waits", n.admission_waits},
                       {"evictions", n.evictions},
                       {"weights_shared_by", wshare}});
    }
    s.makespan = makespan_;
    s.prefill_wait_samples = std::move(waits_);
    s.session_miss_fallbacks = session_misses_;
    s.route_decisions = std::move(route_log_);
    std::vector<double> hops = hop_ms_;
    std::sort(hops.begin(), hops.end());
    const double mean_tok = link_.transfers > 0 ? xfer_bytes_ / double(link_.transfers) : 0.0;
    json dj = {{"nodes", nodes},
               {"clock", opt_.realtime ? "realtime" : "device"},
               {"kv_transfer", {{"transfers", link_.transfers}, {"bytes", xfer_bytes_}, {"device_ms", xfer_ms_},
                                {"gbs", xfer_ms_ > 0 ? xfer_bytes_ / (xfer_ms_ * 1e-3) / 1e9 : 0.0},
                                {"hop_ms_p50", hops.empty() ? 0.0 : hops[hops.size() / 2]},
                                {"mean_hop_bytes", mean_tok}}},
               {"kv_lifecycle", {{"released_tables", released_tables_}, {"released_tokens", released_tokens_},
                                 {"blocks_in_use_at_end", blocks_in_use}, {"coverage_errors", coverage_errors_},
                                 {"evicted_tokens", evicted_tokens_}}},
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
  int max_step_tokens_ = 0, p_step_tokens_ = 0;
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
  std::vector<double> hop_ms_;
  long released_tables_ = 0, released_tokens_ = 0, coverage_errors_ = 0, evicted_tokens_ = 0;
  std::uint64_t seq_ = 0;
  double now_ = 0, makespan_ = 0, think_;
  long session_misses_ = 0;
  // realtime
  Mailbox mb_;
  Clock::time_point t0_{};
  int inflight_steps_ = 0, inflight_copies_ = 0;
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
