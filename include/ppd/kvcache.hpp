// ppd/kvcache.hpp — the KV-cache manager of a node: a paged block pool.
//
// The reference keeps `std::unordered_map<int,long> prefix_cache` per node
// (simulator.cpp:125): token counts only, no capacity. Here every node owns a
// pool of fixed-size blocks (16 tokens, all layers, resident in that node's
// HBM, see ppd_kv_pool_init) and each conversation cached on the node owns a
// block table. Covered tokens always equal the reference's prefix_cache value
// for the conversation; block ids are handed out lowest-free-first so block
// tables are a deterministic function of the event sequence.
#pragma once

#include <cstdint>
#include <map>
#include <set>
#include <stdexcept>
#include <vector>

namespace ppd::kv {

struct BlockTable {
  std::vector<std::int32_t> blocks;
  long tokens = 0;  // covered tokens (== prefix_cache[conv])
};

class BlockPool {
 public:
  BlockPool(int num_blocks = 0, int block_tokens = 16);
  int block_tokens() const { return block_tokens_; }
  int num_blocks() const { return num_blocks_; }
  int free_blocks() const { return num_blocks_ - fresh_ + static_cast<int>(returned_.size()); }
  int used_blocks() const { return num_blocks_ - free_blocks(); }

  // Grow (never shrink) the blocks of `conv` to hold `tokens` positions without
  // changing its covered-token count; throws std::runtime_error("KV pool
  // exhausted ...") when blocks run out.
  const BlockTable& ensure(int conv, long tokens);
  // Sets covered tokens (allocating as needed); reference prefix_cache[conv] = tokens
  const BlockTable& set_tokens(int conv, long tokens);
  const BlockTable* find(int conv) const;
  // blocks `ensure(conv, tokens)` would have to take from the pool
  int blocks_needed(int conv, long tokens) const;
  long tokens(int conv) const;
  void release(int conv);  // returns all blocks of conv to the pool
  const std::map<int, BlockTable>& tables() const { return tables_; }

 private:
  std::int32_t take();
  int num_blocks_;
  int block_tokens_;
  std::int32_t fresh_ = 0;           // ids >= fresh_ were never handed out
  std::set<std::int32_t> returned_;  // released ids (< fresh_), lowest first
  std::map<int, BlockTable> tables_;
};

}  // namespace ppd::kv
