// sched.cpp -- the gate-level scheduler: compiles VeLoPIR's circuits for a shard of
// records into a list of levels; each level is one batched blind-rotate launch plus one batched
// key-switch launch over every independent gate of that level across all records.
//
// Circuits, written from the paper's listings:
//   HomCompLE / HomCompL  alg:HomCompLE, alg:HomCompL; R11 UNSIGNED selects ct2[l-1]
//   HomEQ / HomEqOPT      alg:HomEQ, alg:HomEquiOPT, R14
//   IntV                  alg:InterValid, R12 CLOSED_UPPER, R13 (d = 2 rectangle)
//   CoV / IdM             alg:BB2
//   mask                  alg:HomBitwiseAND, R16
//   aggregation           alg:HomSum or the pairwise tree, R15, R19
// Level assignment is ASAP on the gate DAG.  A MUX (R10) is two blind rotations, each depending on
// the selector and ONE data input, plus one key switch: each half is scheduled as soon as its own inputs
// exist (the data-independent half of every comparator-ladder MUX is hoisted), the key switch when both
// halves are done.  Ciphertexts do not depend on the schedule: every gate is a pure function of its
// inputs and the evaluation key.
#include <algorithm>
#include <cstring>

#include "vlp_internal.h"

namespace vlp {
namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr size_t kMaxRows = size_t{1} << 28;  // rows addressable by a slot id (region << 28 | row)
// A reference to a node may carry NOT (free: the negated ciphertext, O11): bit 31.  A gate folds it into
// its linear form (the input's coefficient changes sign), so no ciphertext is ever materialised for it.
constexpr uint32_t kNeg = 0x80000000u;
inline uint32_t node_of(uint32_t ref) { return ref & ~kNeg; }
inline int sgn(uint32_t ref) { return (ref & kNeg) ? -1 : 1; }

struct LinForm {
  uint32_t k0;
  int8_t ax, ay;
};
constexpr int kOpRefresh = 100;  // R24 refresh bootstrap of a {0, 1/2}-encoded sum: c = x - 1/4
// S2 / R10 linear forms: c = (0, k0) + ax*x + ay*y.
LinForm form(int op) {
  switch (op) {
    case kOpRefresh: return {0xC0000000u, 1, 0};
    case VLP_AND: return {0xE0000000u, 1, 1};
    case VLP_NAND: return {0x20000000u, -1, -1};
    case VLP_OR: return {0x20000000u, 1, 1};
    case VLP_XOR: return {0x40000000u, 2, 2};
    default: return {0xC0000000u, -2, -2};  // XNOR
  }
}

struct Node {
  uint8_t kind;  // 0 leaf, 1 gate, 2 mux, 3 linear sum (R24; in[0] = index into Builder::lin_inputs)
  uint8_t op;
  uint32_t in[3];
  uint32_t level;      // level at which the output exists (0 for leaves; a linear sum: its inputs' level)
  uint32_t h1, h2;     // MUX half levels
  uint32_t slot;       // leaf: fixed slot id; gate: assigned at finalize
  uint8_t tv = 0;      // gate: test vector (0: 1/8, 1: 1/4)
  uint32_t add = 0;    // gate: constant added to b' before the key switch
};

class Builder {
 public:
  std::vector<Node> nodes;
  uint32_t leaf(uint32_t slot_id) {
    nodes.push_back(Node{0, 0, {kNone, kNone, kNone}, 0, 0, 0, slot_id});
    return static_cast<uint32_t>(nodes.size() - 1);
  }
  uint32_t konst(int bit) {  // trivial (0, +-1/8): rows 0 / 1 of the intermediate region (R21)
    uint32_t& c = bit ? one_ : zero_;
    if (c == kNone) c = leaf(slot(kRegMid, bit ? 1 : 0));
    return c;
  }
  uint32_t lvl(uint32_t ref) const { return nodes[node_of(ref)].level; }
  uint32_t gate(int op, uint32_t x, uint32_t y) {
    const uint32_t l = std::max(lvl(x), lvl(y)) + 1;
    nodes.push_back(Node{1, static_cast<uint8_t>(op), {x, y, kNone}, l, 0, 0, kNone});
    return static_cast<uint32_t>(nodes.size() - 1);
  }
  // MUX(c, a, b) = c ? a : b (R10)
  uint32_t mux(uint32_t c, uint32_t a, uint32_t b) {
    const uint32_t h1 = std::max(lvl(c), lvl(a)) + 1;
    const uint32_t h2 = std::max(lvl(c), lvl(b)) + 1;
    nodes.push_back(Node{2, VLP_MUX, {c, a, b}, std::max(h1, h2), h1, h2, kNone});
    return static_cast<uint32_t>(nodes.size() - 1);
  }
  static uint32_t NOT(uint32_t ref) { return ref ^ kNeg; }
  // a gate with a non-default test vector / post-bootstrap constant (R24)
  uint32_t gate_tv(int op, uint32_t x, uint32_t y, uint8_t tv, uint32_t add) {
    const uint32_t g = gate(op, x, y);
    nodes[g].tv = tv;
    nodes[g].add = add;
    return g;
  }
  // R24: sum of {0, 1/2}-encoded ciphertexts (exact, no bootstrap), available in its inputs' level
  uint32_t lin(const std::vector<uint32_t>& refs) {
    uint32_t l = 0;
    for (uint32_t r : refs) l = std::max(l, lvl(r));
    lin_inputs.push_back(refs);
    nodes.push_back(Node{3, 0, {static_cast<uint32_t>(lin_inputs.size() - 1), kNone, kNone}, l, 0, 0, kNone});
    return static_cast<uint32_t>(nodes.size() - 1);
  }
  std::vector<std::vector<uint32_t>> lin_inputs;
  uint32_t AND(uint32_t x, uint32_t y) { return gate(VLP_AND, x, y); }
  uint32_t OR(uint32_t x, uint32_t y) { return gate(VLP_OR, x, y); }
  uint32_t XOR(uint32_t x, uint32_t y) { return gate(VLP_XOR, x, y); }
  uint32_t XNOR(uint32_t x, uint32_t y) { return gate(VLP_XNOR, x, y); }

  // Assign slots (outputs listed in `outs` go to the out region, in order) and emit the levels.  Slot ids
  // hold a 28-bit row (slot()): a schedule with more intermediate rows is refused.
  // Rows are recycled by liveness (unless keep_all): an intermediate is read by the blind rotations of the
  // levels that consume it (a linear sum's inputs right after its level's key switch), so its row is free
  // again from the level after its last reader on; an N-LWE row from the level after its key switch on.
  // `pinned` nodes (the parity-dump rows v_i and the masked payloads) keep their rows.
  int finalize(const std::vector<uint32_t>& outs, Schedule* s, const std::vector<uint32_t>& pinned = {},
               bool keep_all = true) {
    size_t gates = 0;
    for (auto& nd : nodes) gates += nd.kind != 0;  // every non-leaf node owns an intermediate row
    if (gates + 2 > kMaxRows || outs.size() > kMaxRows)
      return fail(VLP_EINVAL, "schedule too large: more than 2^28 ciphertext rows in one region");
    std::vector<uint32_t> out_index(nodes.size(), kNone);
    for (size_t j = 0; j < outs.size(); j++) {
      if (outs[j] & kNeg) return fail(VLP_EINVAL, "internal: a negated reference as a circuit output");
      if (nodes[outs[j]].kind != 0) out_index[outs[j]] = static_cast<uint32_t>(j);
    }
    uint32_t maxl = 0;
    for (auto& nd : nodes)
      if (nd.kind != 0) maxl = std::max(maxl, nd.level);
    // last level reading each node
    constexpr uint32_t kForever = 0xFFFFFFFFu;
    std::vector<uint32_t> death(nodes.size(), 0);
    auto use = [&](uint32_t ref, uint32_t L) {
      uint32_t& d = death[node_of(ref)];
      d = std::max(d, L);
    };
    for (auto& nd : nodes) {
      if (nd.kind == 1) {
        use(nd.in[0], nd.level);
        use(nd.in[1], nd.level);
      } else if (nd.kind == 2) {
        use(nd.in[0], std::max(nd.h1, nd.h2));
        use(nd.in[1], nd.h1);
        use(nd.in[2], nd.h2);
      } else if (nd.kind == 3) {
        for (uint32_t r : lin_inputs[nd.in[0]]) use(r, nd.level);
      }
    }
    for (uint32_t pnode : pinned) death[node_of(pnode)] = kForever;
    // intermediate rows (0, 1 = the trivial constants) and N-LWE rows, level by level
    std::vector<std::vector<uint32_t>> born(maxl + 1), mid_free_at(maxl + 2), nl_free_at(maxl + 2);
    std::vector<std::vector<std::pair<uint32_t, int>>> brs(maxl + 1);  // (node, half) per BR level
    for (uint32_t i = 0; i < nodes.size(); i++) {
      const Node& nd = nodes[i];
      if (nd.kind == 0) continue;
      if (out_index[i] == kNone) born[nd.level].push_back(i);
      if (nd.kind == 1) brs[nd.level].push_back({i, 1});
      if (nd.kind == 2) {
        brs[nd.h1].push_back({i, 1});
        brs[nd.h2].push_back({i, 2});
      }
    }
    std::vector<uint32_t> row1(nodes.size(), kNone), row2(nodes.size(), kNone);
    std::vector<uint32_t> free_mid, free_nl;
    uint32_t mid = 2, nl = 0;
    for (uint32_t L = 1; L <= maxl; L++) {
      for (uint32_t r : mid_free_at[L]) free_mid.push_back(r);
      for (uint32_t r : nl_free_at[L]) free_nl.push_back(r);
      for (auto [i, h] : brs[L]) {
        uint32_t r;
        if (!keep_all && !free_nl.empty()) {
          r = free_nl.back();
          free_nl.pop_back();
        } else {
          r = nl++;
        }
        (h == 2 ? row2 : row1)[i] = r;
        if (nodes[i].level + 1 <= maxl) nl_free_at[nodes[i].level + 1].push_back(r);
      }
      for (uint32_t i : born[L]) {
        uint32_t r;
        if (!keep_all && !free_mid.empty()) {
          r = free_mid.back();
          free_mid.pop_back();
        } else {
          r = mid++;
        }
        nodes[i].slot = slot(kRegMid, r);
        const uint32_t d = std::max(death[i], nodes[i].level);
        if (d != kForever && d + 1 <= maxl) mid_free_at[d + 1].push_back(r);
      }
    }
    for (uint32_t i = 0; i < nodes.size(); i++)
      if (nodes[i].kind != 0 && out_index[i] != kNone) nodes[i].slot = slot(kRegOut, out_index[i]);
    s->levels.assign(maxl, Level{});
    auto sl = [&](uint32_t ref) { return nodes[node_of(ref)].slot; };
    for (uint32_t i = 0; i < nodes.size(); i++) {
      Node& nd = nodes[i];
      if (nd.kind == 1) {
        const LinForm f = form(nd.op);
        const uint32_t row = row1[i];
        s->levels[nd.level - 1].br.push_back(BrJob{sl(nd.in[0]), sl(nd.in[1]), f.k0,
                                                   static_cast<int8_t>(f.ax * sgn(nd.in[0])),
                                                   static_cast<int8_t>(f.ay * sgn(nd.in[1])), nd.tv, row});
        s->levels[nd.level - 1].ks.push_back(KsJob{row, kNone, nd.add, nd.slot});
        s->gates++;
        s->br++;
        s->ks++;
      } else if (nd.kind == 2) {
        const uint32_t r1 = row1[i], r2 = row2[i];
        const uint32_t c = sl(nd.in[0]), a = sl(nd.in[1]), b = sl(nd.in[2]);
        const int sc = sgn(nd.in[0]), sa = sgn(nd.in[1]), sb = sgn(nd.in[2]);
        // BR_N((0,-1/8) + c + a) and BR_N((0,-1/8) - c + b); KS((0,1/8) + u1 + u2)
        s->levels[nd.h1 - 1].br.push_back(BrJob{c, a, 0xE0000000u, static_cast<int8_t>(sc), static_cast<int8_t>(sa), 0, r1});
        s->levels[nd.h2 - 1].br.push_back(BrJob{c, b, 0xE0000000u, static_cast<int8_t>(-sc), static_cast<int8_t>(sb), 0, r2});
        s->levels[nd.level - 1].ks.push_back(KsJob{r1, r2, kMu, nd.slot});
        s->gates++;
        s->br += 2;
        s->ks++;
      } else if (nd.kind == 3) {
        Level& L = s->levels[nd.level - 1];
        const auto& ins = lin_inputs[nd.in[0]];
        L.lin.push_back(LinJob{nd.slot, static_cast<uint32_t>(L.lin_in.size()), static_cast<uint32_t>(ins.size()), 0});
        for (uint32_t r : ins) {
          if (r & kNeg) return fail(VLP_EINVAL, "internal: negated input of a linear sum");
          L.lin_in.push_back(sl(r));
        }
      }
    }
    s->mid_rows = mid;
    s->nlwe_rows = nl;
    s->out_cts = outs.size();
    for (uint32_t o : outs) s->out_slots.push_back(nodes[node_of(o)].slot);  // outputs are never negated refs
    return VLP_OK;
  }

 private:
  uint32_t zero_ = kNone, one_ = kNone;
};

using Word = std::vector<uint32_t>;  // bit ciphertexts, LSB first (R20)

// alg:HomCompLE / alg:HomCompL: ladder init trivial Enc(1) / Enc(0).
uint32_t comp(Builder& B, const Word& c1, const Word& c2, int l, bool le, bool uns) {
  const uint32_t t0 = B.XOR(c1[l - 1], c2[l - 1]);
  uint32_t t2 = B.konst(le ? 1 : 0);
  for (int i = 0; i <= l - 2; i++) {
    const uint32_t t1 = B.XNOR(c1[i], c2[i]);
    t2 = B.mux(t1, t2, c2[i]);
  }
  return B.mux(t0, uns ? c2[l - 1] : c1[l - 1], t2);
}

// Log-depth (parallel-prefix) comparator, VLP_F_PREFIX_COMP (NOT in the paper -- reading
// R23 in DESIGN.md): returns a reference to [c1 > c2] (unsigned).  Bit ranges r = (G, E) with G = [c1 > c2 on
// the range] and E = [c1 == c2 on the range]; leaves G_i = AND(c1_i, NOT c2_i), E_i = XNOR(c1_i, c2_i);
// ranges are paired (r[2k+1] high, r[2k] low) level by level, an unpaired top range passing through:
// G = MUX(H.E, L.G, H.G) (H.G and H.E are exclusive), E = AND(H.E, L.E).  Only the E gates some G needs are
// built.  Depth 1 + ceil(log2 l) instead of l + 1.
uint32_t comp_gt_prefix(Builder& B, const Word& c1, const Word& c2, int l) {
  // tree shape: idx[level] = ranges of that level as (hi child, lo child) indices into the level below
  std::vector<std::vector<std::pair<int, int>>> lev;
  for (int m = l; m > 1; m = (m + 1) / 2) {
    std::vector<std::pair<int, int>> nx;
    for (int k = 0; 2 * k < m; k++) nx.push_back(2 * k + 1 < m ? std::make_pair(2 * k + 1, 2 * k) : std::make_pair(-1, 2 * k));
    lev.push_back(nx);
  }
  // which ranges need E (top-down): a high child always (for its parent's G), a low child iff its parent's E
  std::vector<std::vector<char>> needE(lev.size() + 1);
  needE[0].assign(l, 0);
  for (size_t L = 0; L < lev.size(); L++) needE[L + 1].assign(lev[L].size(), 0);
  for (size_t L = lev.size(); L-- > 0;) {
    for (size_t k = 0; k < lev[L].size(); k++) {
      const auto [hi, lo] = lev[L][k];
      if (hi < 0) {
        needE[L][lo] |= needE[L + 1][k];  // pass-through
      } else {
        needE[L][hi] = 1;
        needE[L][lo] |= needE[L + 1][k];
      }
    }
  }
  std::vector<uint32_t> G(l), E(l, kNone);
  for (int i = 0; i < l; i++) {
    G[i] = B.AND(c1[i], Builder::NOT(c2[i]));
    if (needE[0][i]) E[i] = B.XNOR(c1[i], c2[i]);
  }
  for (size_t L = 0; L < lev.size(); L++) {
    std::vector<uint32_t> g2(lev[L].size()), e2(lev[L].size(), kNone);
    for (size_t k = 0; k < lev[L].size(); k++) {
      const auto [hi, lo] = lev[L][k];
      if (hi < 0) {
        g2[k] = G[lo];
        e2[k] = E[lo];
        continue;
      }
      g2[k] = B.mux(E[hi], G[lo], G[hi]);
      if (needE[L + 1][k]) e2[k] = B.AND(E[hi], E[lo]);
    }
    G.swap(g2);
    E.swap(e2);
  }
  return G[0];
}

// alg:HomEQ and alg:HomEquiOPT.
uint32_t eq(Builder& B, const Word& c1, const Word& c2, int l, bool tree) {
  if (!tree) {
    uint32_t r = B.konst(1);
    for (int i = 0; i < l; i++) r = B.AND(r, B.XNOR(c1[i], c2[i]));
    return r;
  }
  std::vector<uint32_t> t(l);
  for (int i = 0; i < l; i++) t[i] = B.XNOR(c1[i], c2[i]);
  for (int k = 1; k < l; k *= 2)
    for (int i = 0; i < l; i += 2 * k)
      if (i + k < l) t[i] = B.AND(t[i], t[i + k]);
  return t[0];
}

uint32_t validate(Builder& B, const vlp_meta& m, const std::vector<Word>& q, const std::vector<Word>& rec) {
  const int l = static_cast<int>(m.l_I);
  const bool uns = m.flags & VLP_F_UNSIGNED, closed = m.flags & VLP_F_CLOSED_UPPER, tree = m.flags & VLP_F_EQ_TREE;
  const bool prefix = m.flags & VLP_F_PREFIX_COMP;
  // CompLE(a, b) = [a <= b] = NOT [a > b]; CompL(a, b) = [a < b] = [b > a] (prefix form)
  auto cmp = [&](const Word& a, const Word& b, bool le) {
    if (!prefix) return comp(B, a, b, l, le, uns);
    return le ? Builder::NOT(comp_gt_prefix(B, a, b, l)) : comp_gt_prefix(B, b, a, l);
  };
  if (m.mode == VLP_MODE_INTV) {  // alg:InterValid, operand order of P:342-346
    const uint32_t v_xl = cmp(rec[0], q[0], true);
    const uint32_t v_xr = cmp(q[0], rec[1], closed);
    if (m.d == 1) return B.AND(v_xl, v_xr);
    const uint32_t v_yl = cmp(rec[2], q[1], true);
    const uint32_t v_yr = cmp(q[1], rec[3], closed);
    const uint32_t v_x = B.AND(v_xl, v_xr);
    const uint32_t v_y = B.AND(v_yl, v_yr);
    return B.AND(v_x, v_y);
  }
  if (m.mode == VLP_MODE_COV) {  // alg:BB2
    const uint32_t v_x = eq(B, q[0], rec[0], l, tree);
    const uint32_t v_y = eq(B, q[1], rec[1], l, tree);
    return B.AND(v_x, v_y);
  }
  return eq(B, q[0], rec[0], l, tree);  // IdM
}

// R24 (NOT in the paper): linear XOR aggregation.  The masked bits arrive in the {0, 1/2}
// encoding (mask bootstraps with test vector 1/4, then + 1/4), so a sum of ciphertexts is the XOR of their
// bits; groups of kLinGroup consecutive records are summed without bootstrapping (noise grows by
// sqrt(kLinGroup): 8 sigma of margin at 64) and each group sum is refreshed by one bootstrap of x - 1/4 --
// test vector 1/4 (+ 1/4 again) while groups remain, test vector 1/8 for the final result (the standard
// encoding decrypt_result expects).
constexpr size_t kLinGroup = 64;
Word aggregate_linear(Builder& B, std::vector<Word> S, size_t l_S) {
  while (S.size() > kLinGroup) {
    std::vector<Word> up;
    for (size_t g0 = 0; g0 < S.size(); g0 += kLinGroup) {
      Word w(l_S);
      for (size_t j = 0; j < l_S; j++) {
        std::vector<uint32_t> ins;
        for (size_t i = g0; i < std::min(S.size(), g0 + kLinGroup); i++) ins.push_back(S[i][j]);
        const uint32_t t = B.lin(ins);
        w[j] = B.gate_tv(kOpRefresh, t, t, 1, 0x40000000u);
      }
      up.push_back(w);
    }
    S.swap(up);
  }
  Word R(l_S);
  for (size_t j = 0; j < l_S; j++) {
    std::vector<uint32_t> ins;
    for (auto& w : S) ins.push_back(w[j]);
    const uint32_t t = B.lin(ins);
    R[j] = B.gate_tv(kOpRefresh, t, t, 0, 0u);
  }
  return R;
}

// HomSum tree (R15) or serial alg:HomSum; XOR or OR (R19).  Returns the root word.
Word aggregate(Builder& B, std::vector<Word> S, size_t l_S, uint32_t flags) {
  const int op = (flags & VLP_F_OR_REDUCE) ? VLP_OR : VLP_XOR;
  const size_t M = S.size();
  if (flags & VLP_F_SUM_TREE) {
    for (size_t k = 1; k < M; k *= 2)
      for (size_t i = 0; i < M; i += 2 * k)
        if (i + k < M)
          for (size_t j = 0; j < l_S; j++) S[i][j] = B.gate(op, S[i][j], S[i + k][j]);
    return S[0];
  }
  Word R(l_S);
  for (size_t j = 0; j < l_S; j++) R[j] = B.konst(0);
  for (size_t i = 0; i < M; i++)
    for (size_t j = 0; j < l_S; j++) R[j] = B.gate(op, R[j], S[i][j]);
  return R;
}

}  // namespace

int compile_velopir(const vlp_meta& m, size_t first, size_t count, Schedule* s, uint32_t nq) {
  if (int rc = check_meta(&m)) return rc;
  if (count == 0 || first + count > m.M) return fail(VLP_EINVAL, "bad record range");
  if (nq < 1 || nq > 4096) return fail(VLP_EINVAL, "query count must be in [1, 4096]");
  if ((m.flags & VLP_F_PREFIX_COMP) && !(m.flags & VLP_F_UNSIGNED))
    return fail(VLP_EINVAL, "the prefix comparator is unsigned only (VLP_F_UNSIGNED)");
  const bool linear = m.flags & VLP_F_LINEAR_SUM;
  if (linear && (m.flags & VLP_F_OR_REDUCE)) return fail(VLP_EINVAL, "linear aggregation computes XOR only");
  Builder B;
  const size_t l = m.l_I, W = record_words(m), QW = query_words(m), per = W * l + m.l_S;
  if (count * per > kMaxRows || static_cast<size_t>(nq) * QW * l > kMaxRows)
    return fail(VLP_EINVAL, "shard too large: more than 2^28 input ciphertexts");
  // the shard's record ciphertexts are shared by all nq queries (multi-query packing)
  std::vector<std::vector<Word>> recs(count, std::vector<Word>(W, Word(l)));
  std::vector<Word> pays(count, Word(m.l_S));
  for (size_t r = 0; r < count; r++) {
    const uint32_t base = static_cast<uint32_t>(r * per);
    for (size_t k = 0; k < W; k++)
      for (size_t j = 0; j < l; j++) recs[r][k][j] = B.leaf(slot(kRegIn1, base + static_cast<uint32_t>(k * l + j)));
    for (size_t j = 0; j < m.l_S; j++) pays[r][j] = B.leaf(slot(kRegIn1, base + static_cast<uint32_t>(W * l + j)));
  }
  Word outs;
  std::vector<uint32_t> vs(count);
  std::vector<Word> masked0;
  for (uint32_t qi = 0; qi < nq; qi++) {
    std::vector<Word> q(QW, Word(l));
    for (size_t w = 0; w < QW; w++)
      for (size_t j = 0; j < l; j++)
        q[w][j] = B.leaf(slot(kRegIn0, static_cast<uint32_t>((qi * QW + w) * l + j)));
    std::vector<Word> masked(count);
    for (size_t r = 0; r < count; r++) {  // alg:VeLoPIR record loop
      const uint32_t v = validate(B, m, q, recs[r]);
      if (qi == 0) vs[r] = v;
      masked[r].resize(m.l_S);
      for (size_t j = 0; j < m.l_S; j++)  // alg:HomBitwiseAND (R16); R24: into the {0, 1/2} encoding
        masked[r][j] = linear ? B.gate_tv(VLP_AND, v, pays[r][j], 1, 0x40000000u) : B.AND(v, pays[r][j]);
    }
    const Word root = linear ? aggregate_linear(B, masked, m.l_S) : aggregate(B, masked, m.l_S, m.flags);
    outs.insert(outs.end(), root.begin(), root.end());
    if (qi == 0) masked0 = masked;
  }
  std::vector<uint32_t> pinned(vs.begin(), vs.end());  // parity-dump rows of the first query
  for (auto& w : masked0) pinned.insert(pinned.end(), w.begin(), w.end());
  if (int rc = B.finalize(outs, s, pinned, m.flags & VLP_F_KEEP_ALL)) return rc;
  s->in0_cts = static_cast<uint64_t>(nq) * QW * l;
  s->in1_cts = count * per;
  s->l_S = m.l_S;
  for (size_t r = 0; r < count; r++) {  // parity dumps: the first query's nodes
    s->v_rows.push_back(B.nodes[vs[r]].slot);
    for (size_t j = 0; j < m.l_S; j++) s->mask_rows.push_back(B.nodes[masked0[r][j]].slot);
  }
  return VLP_OK;
}

int compile_gates(int op, size_t count, Schedule* s) {
  if (op < VLP_AND || op > VLP_MUX) return fail(VLP_EINVAL, "bad gate op");
  if (count == 0 || count >= (1u << 27)) return fail(VLP_EINVAL, "bad gate count");
  Builder B;
  std::vector<uint32_t> outs(count);
  for (size_t i = 0; i < count; i++) {
    const uint32_t a = B.leaf(slot(kRegIn0, static_cast<uint32_t>(i)));
    const uint32_t b = B.leaf(slot(kRegIn1, static_cast<uint32_t>(i)));
    if (op == VLP_MUX)
      outs[i] = B.mux(a, b, B.leaf(slot(kRegIn1, static_cast<uint32_t>(count + i))));
    else
      outs[i] = B.gate(op, a, b);
  }
  if (int rc = B.finalize(outs, s)) return rc;
  s->in0_cts = count;
  s->in1_cts = op == VLP_MUX ? 2 * count : count;
  return VLP_OK;
}

int compile_combine(const vlp_meta& m, uint32_t G, Schedule* s) {
  if (int rc = check_meta(&m)) return rc;
  if (G < 1 || G > 65536 || (G & (G - 1))) return fail(VLP_EINVAL, "G must be a power of two <= 65536");
  Builder B;
  std::vector<Word> S(G, Word(m.l_S));
  for (uint32_t g = 0; g < G; g++)
    for (size_t j = 0; j < m.l_S; j++) S[g][j] = B.leaf(slot(kRegIn0, static_cast<uint32_t>(g * m.l_S + j)));
  vlp_meta mm = m;
  mm.flags |= VLP_F_SUM_TREE;  // shard roots combine with the same pairing (R15)
  const Word root = aggregate(B, S, m.l_S, mm.flags);
  if (int rc = B.finalize(root, s)) return rc;
  s->in0_cts = static_cast<uint64_t>(G) * m.l_S;
  s->l_S = m.l_S;
  return VLP_OK;
}

}  // namespace vlp
