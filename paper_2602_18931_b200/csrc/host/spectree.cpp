// Flat-pool SpecTree; semantics follow spectree.hpp:63-323 line by line (cited per method).
#include "spectree.hpp"

#include <algorithm>

namespace wsb {

void SpecTree::reset(std::size_t max_nodes) {
  max_nodes_ = max_nodes;
  for (auto s : live_) slots_[s].children.clear();
  if (slots_.size() < max_nodes + 16) slots_.resize(max_nodes + 16);
  free_.clear();
  for (std::size_t i = slots_.size(); i-- > 0;) free_.push_back(static_cast<std::uint32_t>(i));
  id2slot_.assign(1, -1);
  live_.clear();
  root_children_.clear();
  next_id_ = 1;
  committed_len_ = 0;
  depth_ = 0;
}

NodeId SpecTree::find_child(NodeId parent, TokenId token) const {
  const std::vector<NodeId>& kids = parent == kRootId ? root_children_ : node(parent).children;
  for (NodeId c : kids)
    if (node(c).token == token) return c;
  return kRootId;
}

bool SpecTree::resolve_path(const TokenId* toks, std::size_t n, NodeId* out) const {
  NodeId cur = kRootId;
  for (std::size_t i = 0; i < n; ++i) {
    NodeId next = find_child(cur, toks[i]);
    if (next == kRootId) return false;
    cur = next;
  }
  *out = cur;
  return true;
}

void SpecTree::path_tokens(NodeId id, std::vector<TokenId>& out) const {
  out.clear();
  for (NodeId cur = id; cur != kRootId; cur = node(cur).parent) out.push_back(node(cur).token);
  std::reverse(out.begin(), out.end());
}

// spectree.hpp:111-146
bool SpecTree::append(NodeId parent, const CandIn* cands, std::size_t n, Origin origin) {
  if (parent != kRootId && !contains(parent)) return false;
  for (std::size_t i = 0; i < n; ++i) {
    const CandIn& c = cands[i];
    if (find_child(parent, c.token) != kRootId) continue;  // dedup: existing node reused
    const NodeId id = next_id_++;
    if (free_.empty()) {
      std::size_t old = slots_.size();
      slots_.resize(old * 2 + 16);
      for (std::size_t s = slots_.size(); s-- > old;) free_.push_back(static_cast<std::uint32_t>(s));
    }
    const std::uint32_t slot = free_.back();
    free_.pop_back();
    if (id2slot_.size() <= id) id2slot_.resize(static_cast<std::size_t>(id) * 2 + 64, -1);
    id2slot_[id] = static_cast<std::int32_t>(slot);
    Node& nd = slots_[slot];
    nd.id = id;
    nd.token = c.token;
    nd.prob = c.prob;
    nd.entropy = c.entropy;
    nd.parent = parent;
    nd.origin = origin;
    nd.children.clear();
    nd.live_pos = static_cast<std::uint32_t>(live_.size());
    live_.push_back(slot);
    if (parent == kRootId) {
      nd.depth = 1;
      nd.path_prob = c.prob;
      root_children_.push_back(id);
    } else {
      Node& p = mnode(parent);
      nd.depth = p.depth + 1;
      nd.path_prob = p.path_prob * c.prob;
      p.children.push_back(id);
    }
    depth_ = std::max(depth_, nd.depth);
  }
  evict_over_capacity();
  return true;
}

// spectree.hpp:244-253: drop the last-ranked leaf until within capacity.
void SpecTree::evict_over_capacity() {
  while (live_.size() > max_nodes_) {
    const Node* worst = nullptr;
    for (std::uint32_t s : live_) {
      const Node& n = slots_[s];
      if (!n.children.empty()) continue;
      if (!worst || rank_before(*worst, n)) worst = &n;
    }
    erase_leaf(worst->id);
  }
}

// spectree.hpp:255-262
void SpecTree::erase_leaf(NodeId id) {
  const NodeId parent = node(id).parent;
  std::vector<NodeId>& kids = parent == kRootId ? root_children_ : mnode(parent).children;
  kids.erase(std::find(kids.begin(), kids.end(), id));
  free_node(id);
  recompute_depth();
}

void SpecTree::free_node(NodeId id) {
  const std::uint32_t slot = static_cast<std::uint32_t>(id2slot_[id]);
  id2slot_[id] = -1;
  Node& n = slots_[slot];
  const std::uint32_t pos = n.live_pos;
  const std::uint32_t last = live_.back();
  live_[pos] = last;
  slots_[last].live_pos = pos;
  live_.pop_back();
  n.children.clear();
  free_.push_back(slot);
}

// spectree.hpp:264-268
void SpecTree::clear_nodes() {
  for (std::uint32_t s : live_) {
    id2slot_[slots_[s].id] = -1;
    slots_[s].children.clear();
    free_.push_back(s);
  }
  live_.clear();
  root_children_.clear();
  depth_ = 0;
}

// spectree.hpp:154-179
bool SpecTree::prune(const Validation& v) {
  NodeId cur = kRootId;
  bool complete = true;
  const std::size_t walk = v.accepted.size() + 1;
  for (std::size_t i = 0; i < walk; ++i) {
    const TokenId t = i < v.accepted.size() ? v.accepted[i] : v.bonus;
    NodeId next = find_child(cur, t);
    if (next == kRootId) {
      complete = false;
      break;
    }
    cur = next;
  }
  committed_len_ += walk;
  if (complete)
    reroot_at(cur);
  else
    clear_nodes();
  return complete;
}

// spectree.hpp:270-280: keep only the survivor's subtree; its children become root children.
void SpecTree::reroot_at(NodeId survivor) {
  if (mark_.size() < slots_.size()) mark_.resize(slots_.size());
  for (std::uint32_t s : live_) mark_[s] = 0;
  scratch_.clear();
  scratch_.push_back(survivor);
  while (!scratch_.empty()) {
    NodeId id = scratch_.back();
    scratch_.pop_back();
    const Node& n = node(id);
    mark_[static_cast<std::size_t>(id2slot_[id])] = 1;
    for (NodeId c : n.children) scratch_.push_back(c);
  }
  root_children_ = node(survivor).children;
  mark_[static_cast<std::size_t>(id2slot_[survivor])] = 0;
  // free every unmarked live node (iterate a snapshot: free_node edits live_)
  std::vector<std::uint32_t> snapshot(live_);
  for (std::uint32_t s : snapshot)
    if (!mark_[s]) free_node(slots_[s].id);
  depth_ = 0;
  for (NodeId c : root_children_) rebase(c, kRootId, 0, 1.0);
}

// spectree.hpp:288-296
void SpecTree::rebase(NodeId id, NodeId parent, std::uint32_t parent_depth, double parent_pp) {
  Node& n = mnode(id);
  n.parent = parent;
  n.depth = parent_depth + 1;
  n.path_prob = parent_pp * n.prob;
  depth_ = std::max(depth_, n.depth);
  for (NodeId c : n.children) rebase(c, id, n.depth, n.path_prob);
}

// spectree.hpp:298-301
void SpecTree::recompute_depth() {
  depth_ = 0;
  for (std::uint32_t s : live_) depth_ = std::max(depth_, slots_[s].depth);
}

// spectree.hpp:184-193: partial selection of the s best-ranked leaves.
std::size_t SpecTree::frontier(std::size_t s, NodeId* out) const {
  if (live_.empty()) {
    out[0] = kRootId;
    return 1;
  }
  if (s > 64) {  // rare: full sort (spectree.hpp:189-191)
    std::vector<const Node*> leaves;
    for (std::uint32_t slot : live_)
      if (slots_[slot].children.empty()) leaves.push_back(&slots_[slot]);
    std::sort(leaves.begin(), leaves.end(),
              [](const Node* a, const Node* b) { return rank_before(*a, *b); });
    std::size_t cnt = std::min(s, leaves.size());
    for (std::size_t i = 0; i < cnt; ++i) out[i] = leaves[i]->id;
    return cnt;
  }
  std::size_t cnt = 0;
  const Node* best[64];
  const std::size_t cap = s;
  for (std::uint32_t slot : live_) {
    const Node& n = slots_[slot];
    if (!n.children.empty()) continue;
    if (cnt == cap && !rank_before(n, *best[cnt - 1])) continue;
    std::size_t i = cnt < cap ? cnt++ : cap - 1;
    while (i > 0 && rank_before(n, *best[i - 1])) {
      best[i] = best[i - 1];
      --i;
    }
    best[i] = &n;
  }
  for (std::size_t i = 0; i < cnt; ++i) out[i] = best[i]->id;
  return cnt;
}

// spectree.hpp:202-217
bool SpecTree::best_path(std::uint32_t k, NodeId* ids, TokenId* toks) const {
  if (depth_ < k) return false;
  const Node* best = nullptr;
  for (std::uint32_t slot : live_) {
    const Node& n = slots_[slot];
    if (n.depth != k) continue;
    if (!best || rank_before(n, *best)) best = &n;
  }
  if (!best) return false;
  for (NodeId cur = best->id; cur != kRootId;) {
    const Node& n = node(cur);
    ids[n.depth - 1] = n.id;
    toks[n.depth - 1] = n.token;
    cur = n.parent;
  }
  return true;
}

}  // namespace wsb
