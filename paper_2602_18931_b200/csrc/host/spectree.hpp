// Speculative token tree — same contract as the reference SpecTree (spectree.hpp:63-323):
// content-addressed children (dedup by token), capacity eviction of the worst leaf,
// prune = walk accepted+bonus then reroot at the survivor or clear, frontier(s) and
// best_path(k) ranked by (path_prob desc, depth asc, id asc). Storage is a flat slot pool
// with an id→slot table (ids are never reused within a request), so every query is a
// linear scan over <= max_nodes live nodes instead of std::map walks.
#pragma once

#include "common.hpp"

#include <cstddef>
#include <cstdint>
#include <vector>

namespace wsb {

class SpecTree {
 public:
  struct Node {
    NodeId id = 0;
    TokenId token = 0;
    double prob = 0.0;
    double entropy = 0.0;
    double path_prob = 0.0;
    NodeId parent = kRootId;
    std::uint32_t depth = 0;
    Origin origin = Origin::worker;
    std::uint32_t live_pos = 0;     // index in live_
    std::vector<NodeId> children;   // insertion order (find_child scans it)
  };

  explicit SpecTree(std::size_t max_nodes = 64) { reset(max_nodes); }

  void reset(std::size_t max_nodes);

  std::uint64_t committed_len() const { return committed_len_; }
  std::size_t node_count() const { return live_.size(); }
  std::uint32_t depth() const { return depth_; }
  bool empty() const { return live_.empty(); }
  bool contains(NodeId id) const {
    return id != kRootId && id < id2slot_.size() && id2slot_[id] >= 0;
  }
  const Node& node(NodeId id) const { return slots_[static_cast<std::size_t>(id2slot_[id])]; }

  // spectree.hpp:75-77
  std::uint64_t extension_position(NodeId id) const {
    return id == kRootId ? committed_len_ : committed_len_ + node(id).depth;
  }

  // spectree.hpp:87-95; returns false when the path leaves the tree.
  bool resolve_path(const TokenId* toks, std::size_t n, NodeId* out) const;

  // spectree.hpp:98-104 (root child first, id inclusive).
  void path_tokens(NodeId id, std::vector<TokenId>& out) const;

  // spectree.hpp:111-146: false when the parent is unknown (stale speculation).
  bool append(NodeId parent, const CandIn* cands, std::size_t n, Origin origin);

  // spectree.hpp:154-179; returns true when the walk stayed in the tree (survivor kept).
  bool prune(const Validation& v);

  // spectree.hpp:184-193; writes up to s ids to out, returns the count.
  std::size_t frontier(std::size_t s, NodeId* out) const;

  // spectree.hpp:202-217; false when the tree is not k deep.
  bool best_path(std::uint32_t k, NodeId* ids, TokenId* toks) const;

 private:
  Node& mnode(NodeId id) { return slots_[static_cast<std::size_t>(id2slot_[id])]; }
  NodeId find_child(NodeId parent, TokenId token) const;
  // spectree.hpp:238-242
  static bool rank_before(const Node& a, const Node& b) {
    if (a.path_prob != b.path_prob) return a.path_prob > b.path_prob;
    if (a.depth != b.depth) return a.depth < b.depth;
    return a.id < b.id;
  }
  void evict_over_capacity();
  void erase_leaf(NodeId id);
  void free_node(NodeId id);
  void clear_nodes();
  void reroot_at(NodeId survivor);
  void rebase(NodeId id, NodeId parent, std::uint32_t parent_depth, double parent_pp);
  void recompute_depth();

  std::vector<Node> slots_;
  std::vector<std::uint32_t> free_;
  std::vector<std::int32_t> id2slot_;
  std::vector<std::uint32_t> live_;  // live slot indices (unordered)
  std::vector<NodeId> root_children_;
  std::vector<NodeId> scratch_;
  std::vector<unsigned char> mark_;
  NodeId next_id_ = 1;
  std::uint64_t committed_len_ = 0;
  std::uint32_t depth_ = 0;
  std::size_t max_nodes_ = 64;
};

}  // namespace wsb
