// kvcache.cpp — deterministic paged block allocator (lowest free id first).
#include "ppd/kvcache.hpp"

#include <string>

namespace ppd::kv {

BlockPool::BlockPool(int num_blocks, int block_tokens) : num_blocks_(num_blocks), block_tokens_(block_tokens) {
  if (block_tokens < 1) throw std::invalid_argument("block_tokens must be >= 1");
  if (num_blocks < 0) throw std::invalid_argument("num_blocks must be >= 0");
}

std::int32_t BlockPool::take() {
  if (!returned_.empty()) {
    std::int32_t b = *returned_.begin();
    returned_.erase(returned_.begin());
    return b;
  }
  if (fresh_ >= num_blocks_)
    throw std::runtime_error("KV pool exhausted: " + std::to_string(num_blocks_) + " blocks of " +
                             std::to_string(block_tokens_) + " tokens in use");
  return fresh_++;
}

const BlockTable& BlockPool::ensure(int conv, long tokens) {
  BlockTable& t = tables_[conv];
  const std::size_t need = static_cast<std::size_t>((tokens + block_tokens_ - 1) / block_tokens_);
  while (t.blocks.size() < need) t.blocks.push_back(take());
  return t;
}

const BlockTable& BlockPool::set_tokens(int conv, long tokens) {
  const BlockTable& t = ensure(conv, tokens);
  tables_[conv].tokens = tokens;
  return t;
}

const BlockTable* BlockPool::find(int conv) const {
  auto it = tables_.find(conv);
  return it == tables_.end() ? nullptr : &it->second;
}

int BlockPool::blocks_needed(int conv, long tokens) const {
  const long need = (tokens + block_tokens_ - 1) / block_tokens_;
  const BlockTable* t = find(conv);
  const long have = t ? static_cast<long>(t->blocks.size()) : 0;
  return need > have ? static_cast<int>(need - have) : 0;
}

long BlockPool::tokens(int conv) const {
  const BlockTable* t = find(conv);
  return t ? t->tokens : 0;
}

void BlockPool::release(int conv) {
  auto it = tables_.find(conv);
  if (it == tables_.end()) return;
  for (std::int32_t b : it->second.blocks) returned_.insert(b);
  tables_.erase(it);
}

}  // namespace ppd::kv
