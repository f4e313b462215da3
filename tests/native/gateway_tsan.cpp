// ThreadSanitizer stress of the gateway's concurrency (SURVEY §5 "race
// detection": TSAN on the host scheduler). Built by tests/test_gateway.py with
// -fsanitize=thread against engine/gateway.cpp and its host dependencies.
//
// One loopback server; 6 GPU workers register and heartbeat on their own
// threads (WorkerAgent); 8 client threads route 300 turns each over their own
// connections while an admin thread prunes, evicts sessions and reads stats
// through the in-process API. Exit 0 iff every reply is well-formed and every
// follow-up turn of a conversation lands on the backend its first turn pinned.
#include <atomic>
#include <cstdio>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include <json.hpp>

#include "ppd/gateway.hpp"

using nlohmann::json;
using namespace ppd;

int main() {
  gateway::Gateway gw(routing::RoutingPolicy::static_policy(1.0));
  std::atomic<bool> stop{false};
  std::atomic<int> port{0};
  std::thread srv([&] { gateway::serve_tcp(gw, 0, stop, &port); });
  while (port.load() == 0) std::this_thread::sleep_for(std::chrono::milliseconds(1));

  std::vector<std::unique_ptr<gateway::WorkerAgent>> workers;
  workers.push_back(std::make_unique<gateway::WorkerAgent>(port.load(), 'P', 0, "gpu0", 0.01));
  workers.push_back(std::make_unique<gateway::WorkerAgent>(port.load(), 'P', 1, "gpu1", 0.01));
  for (int g = 2; g < 6; ++g)
    workers.push_back(std::make_unique<gateway::WorkerAgent>(port.load(), 'D', g, "gpu" + std::to_string(g), 0.01));

  std::atomic<int> bad{0};
  std::vector<std::thread> clients;
  for (int c = 0; c < 8; ++c) {
    clients.emplace_back([&, c] {
      gateway::Connection conn(port.load());
      std::map<std::string, int> pin;
      for (int i = 0; i < 300; ++i) {
        const std::string conv = "t" + std::to_string(c) + "-c" + std::to_string(i % 17);
        const bool follow = pin.count(conv) > 0;
        const json r = json::parse(conn.call(json{{"kind", "route"},
                                                   {"conv_first_message", conv},
                                                   {"turn_index", follow ? 2 : 1},
                                                   {"new_input_tokens", 256},
                                                   {"cached_context_tokens", follow ? 512 : 0},
                                                   {"target_output_tokens", 64}}
                                                  .dump(),
                                              i % 3 == 0 ? 5 : 0));
        if (!r.value("ok", false) || !r.contains("decode_gpu")) {
          ++bad;
          continue;
        }
        const int d = r.at("decode_backend").get<int>();
        if (follow && (d != pin[conv] || r.at("target") != "D_local")) ++bad;
        if (!follow) pin[conv] = d;
      }
    });
  }
  std::thread admin([&] {
    for (int i = 0; i < 200; ++i) {
      gw.registry().prune_dead(1e18, 1e30);  // prunes nothing, takes the locks
      gw.sessions().evict_expired(0.0, 1e30);
      (void)gw.stats();
      (void)gw.registry().snapshot();
      std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
  });
  for (auto& t : clients) t.join();
  admin.join();
  long beats = 0;
  for (auto& w : workers) beats += w->heartbeats();
  workers.clear();
  stop.store(true);
  srv.join();
  const auto st = gw.stats();
  std::printf("{\"bad\": %d, \"queries\": %ld, \"heartbeats\": %ld, \"backends\": %ld}\n", bad.load(), st.queries,
              beats, st.backends);
  return bad.load() == 0 && st.queries == 8 * 300 ? 0 : 1;
}
