// pf_symbolic.hpp — symbolic analysis of one sparse symmetric system (a
// subdomain saddle K_s, an interior block K_II, or the mortar Gram matrix
// G G^T): nested-dissection ordering, elimination tree, supernodes, and the
// two-level task schedule the device sweeps run on:
//   * "leaf tasks": maximal etree subtrees below a weight cap, one warp each;
//     their columns are contiguous and their updates to ancestor rows go to a
//     private contribution buffer (deterministic, no atomics);
//   * "top": the remaining ancestors, one CTA per problem, which folds the
//     contribution buffers in fixed task order.
// Columns are renumbered so that every task is a contiguous range and the top
// part is the suffix (a topological order of the supernodal tree).
// Factor storage per supernode: strict lower trapezoid, column-major, column j
// holding rows j+1..m-1 (the unit diagonal is implicit, D stored separately).
#pragma once

#include <functional>

#include "pf_common.hpp"
#include "pf_layout.hpp"

namespace pf {

struct SymFactor {
  int n = 0;
  std::vector<int> perm, iperm;  // position -> natural, natural -> position
  int nsn = 0;
  std::vector<int> sn_col0, sn_ncol, sn_nrow, sn_task;  // sn_task: owning task or -1 (top)
  std::vector<long long> sn_rowoff, sn_valoff;
  std::vector<int> rows;   // row positions per supernode (first ncol = own columns)
  std::vector<int> slot;   // parallel to rows: slot in the task (or top) workspace
  long long nval = 0;
  int ntask = 0;             // all tasks, ordered by level
  std::vector<int> task_sn0, task_sn1, task_c0, task_c1, task_cboff, task_cblen, task_level;
  std::vector<int> level_ptr;  // tasks of level l: [level_ptr[l], level_ptr[l+1])
  int nlevel = 0;              // level 0: warp tasks; 1..nlevel-2: CTA tasks; nlevel-1: root tasks
  std::vector<int> cb_rows;    // positions (ancestor rows of each task)
  std::vector<int> fold_ptr, fold_idx;  // per column: contributions (CB indices) from lower-level tasks
  int top_sn0 = 0, top_c0 = 0; // first supernode / column of the root level
  int max_task_ws = 0;         // max (c1-c0)+cblen over level-0 tasks
  std::vector<int> level_ws;   // max (c1-c0)+cblen per level
  long long flops_factor = 0;
};

/// Nested dissection on half-cell grid coordinates; separators are the
/// vertices of a cut line plus any left vertex adjacent to the right side.
inline void nd_rec(std::vector<int>& ids, const std::vector<std::array<int, 2>>& ic, const Csr& A,
                   std::vector<uint8_t>& side, std::vector<int>& out, int leaf) {
  if ((int)ids.size() <= leaf) {
    std::sort(ids.begin(), ids.end());
    out.insert(out.end(), ids.begin(), ids.end());
    return;
  }
  int lo[2] = {INT32_MAX, INT32_MAX}, hi[2] = {INT32_MIN, INT32_MIN};
  for (int d : ids)
    for (int a = 0; a < 2; ++a) lo[a] = std::min(lo[a], ic[d][a]), hi[a] = std::max(hi[a], ic[d][a]);
  const int first = (hi[0] - lo[0] >= hi[1] - lo[1]) ? 0 : 1;
  for (int attempt = 0; attempt < 2; ++attempt) {
    const int ax = attempt == 0 ? first : 1 - first;
    if (hi[ax] - lo[ax] < 2) continue;
    std::vector<int> v;
    v.reserve(ids.size());
    for (int d : ids) v.push_back(ic[d][ax]);
    std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end());
    const int med = v[v.size() / 2];
    // among vertex lines (even) near the median, take the one crossing the
    // fewest dofs (for the multiplier graph this avoids cutting along an
    // interface line)
    std::sort(v.begin(), v.end());
    const int span = std::max(2, (hi[ax] - lo[ax]) / 8);
    int c = INT32_MIN;
    long long best = -1;
    for (int cand = med - span; cand <= med + span; ++cand) {
      if (cand % 2 || cand <= lo[ax] || cand >= hi[ax]) continue;
      const long long cnt = std::upper_bound(v.begin(), v.end(), cand) - std::lower_bound(v.begin(), v.end(), cand);
      const long long left = std::lower_bound(v.begin(), v.end(), cand) - v.begin();
      const long long imb = std::llabs(2 * left + cnt - (long long)v.size());
      const long long score = cnt * 4 * (long long)v.size() / std::max<long long>(1, hi[ax] - lo[ax]) + imb;
      if (best < 0 || score < best) best = score, c = cand;
    }
    if (c == INT32_MIN) {
      c = med + (med % 2 ? 1 : 0);
      c = std::max(lo[ax] + 1, std::min(hi[ax] - 1, c));
    }
    std::vector<int> L, R, S;
    for (int d : ids) (ic[d][ax] < c ? L : ic[d][ax] > c ? R : S).push_back(d);
    for (int d : R) side[d] = 1;
    std::vector<int> L2;
    L2.reserve(L.size());
    for (int d : L) {
      bool cross = false;
      for (int q = A.ptr[d]; q < A.ptr[d + 1] && !cross; ++q) cross = side[A.col[q]] == 1;
      (cross ? S : L2).push_back(d);
    }
    for (int d : R) side[d] = 0;
    if (L2.empty() && R.empty()) continue;
    nd_rec(L2, ic, A, side, out, leaf);
    nd_rec(R, ic, A, side, out, leaf);
    std::sort(S.begin(), S.end());
    out.insert(out.end(), S.begin(), S.end());
    return;
  }
  std::sort(ids.begin(), ids.end());
  out.insert(out.end(), ids.begin(), ids.end());
}

/// Build the symbolic factor of symmetric pattern A (natural order).
/// task_cap: maximum packed-value weight of one leaf task (0 = no tasks).
/// Symbolic analysis.  Default: nested dissection of all of A.  With
/// `root_last` (natural indices, in order), those columns are eliminated last
/// as ONE dense root supernode and nested dissection orders the rest (the
/// bordered dual-operator factorisation, pf_dual.hpp).
inline SymFactor analyse(const Csr& A, const std::vector<std::array<int, 2>>& ic, long long task_cap,
                         int ws_cap = 640, double amalg_zero_frac = 0.15, int amalg_small = 16, int leaf = 48,
                         const std::vector<int>* root_last = nullptr) {
  SymFactor F;
  const int n = A.nr;
  F.n = n;
  std::vector<int> order;
  const int root_cols = root_last ? (int)root_last->size() : 0;
  {
    std::vector<int> ids;
    std::vector<char> in_root(n, 0);
    if (root_last)
      for (int r : *root_last) in_root[r] = 1;
    for (int i = 0; i < n; ++i)
      if (!in_root[i]) ids.push_back(i);
    std::vector<uint8_t> side(n, 0);
    order.reserve(n);
    nd_rec(ids, ic, A, side, order, leaf);
    if (root_last) order.insert(order.end(), root_last->begin(), root_last->end());
  }
  std::vector<int> ip(n);
  for (int k = 0; k < n; ++k) ip[order[k]] = k;
  // permuted strictly-lower adjacency: for column k, rows i > k
  std::vector<std::vector<int>> lower(n);
  for (int r = 0; r < n; ++r)
    for (int q = A.ptr[r]; q < A.ptr[r + 1]; ++q) {
      const int i = ip[r], j = ip[A.col[q]];
      if (i > j) lower[j].push_back(i);
    }
  // elimination tree (Liu) using row view: for row k, entries j < k
  std::vector<std::vector<int>> upper(n);  // upper[k] = cols j < k with A(k,j) != 0
  for (int j = 0; j < n; ++j)
    for (int i : lower[j]) upper[i].push_back(j);
  std::vector<int> parent(n, -1), anc(n, -1);
  for (int k = 0; k < n; ++k)
    for (int j : upper[k]) {
      int r = j;
      while (anc[r] != -1 && anc[r] != k) {
        const int nx = anc[r];
        anc[r] = k;
        r = nx;
      }
      if (anc[r] == -1) {
        anc[r] = k;
        parent[r] = k;
      }
    }
  // column counts via row-subtree traversal
  std::vector<int> cc(n, 1), flag(n, -1);
  for (int k = 0; k < n; ++k) {
    flag[k] = k;
    for (int j : upper[k])
      for (int i = j; flag[i] != k; i = parent[i]) {
        cc[i]++;
        flag[i] = k;
      }
  }
  // fundamental supernodes
  std::vector<int> nchild(n, 0);
  for (int j = 0; j < n; ++j)
    if (parent[j] >= 0) nchild[parent[j]]++;
  std::vector<int> sn_of(n), s0;
  for (int j = 0; j < n; ++j) {
    bool join = j > 0 && parent[j - 1] == j && cc[j - 1] == cc[j] + 1 && nchild[j] == 1;
    if (root_cols) {
      if (j == n - root_cols) join = false;  // the root block starts a supernode ...
      else if (j > n - root_cols) join = true;  // ... and is one supernode
    }
    if (!join) s0.push_back(j);
    sn_of[j] = (int)s0.size() - 1;
  }
  int ns = (int)s0.size();
  s0.push_back(n);
  // supernodal parent and structures
  std::vector<int> sparent(ns, -1);
  for (int s = 0; s < ns; ++s) {
    const int last = s0[s + 1] - 1;
    if (parent[last] >= 0) sparent[s] = sn_of[parent[last]];
  }
  std::vector<std::vector<int>> schild(ns);
  for (int s = 0; s < ns; ++s)
    if (sparent[s] >= 0) schild[sparent[s]].push_back(s);
  std::vector<std::vector<int>> st(ns);
  std::vector<int> mark(n, -1);
  for (int s = 0; s < ns; ++s) {
    const int c0 = s0[s], c1 = s0[s + 1];
    std::vector<int>& R = st[s];
    for (int c = c0; c < c1; ++c) R.push_back(c), mark[c] = s;
    for (int c = c0; c < c1; ++c)
      for (int r : lower[c])
        if (r >= c1 && mark[r] != s) mark[r] = s, R.push_back(r);
    for (int ch : schild[s])
      for (int r : st[ch])
        if (r >= c1 && mark[r] != s) mark[r] = s, R.push_back(r);
    std::sort(R.begin() + (c1 - c0), R.end());
  }
  // ---- relaxed amalgamation: absorb a child into its parent when the child's
  // columns immediately precede the parent's and the merged block is small or
  // adds few explicit zeros (fewer, wider supernodes for the device sweeps) ----
  if (amalg_zero_frac > 0.0) {
    std::vector<int> head(ns);  // first supernode index of the merged group ending at s
    std::vector<long long> nv(ns);
    auto val_count = [](long long n, long long m) { return n * m - n * (n + 1) / 2; };
    std::vector<int> c0(ns), nrow(ns);  // current first column and row count of group ending at s
    std::vector<long long> zeros(ns, 0);
    for (int s = 0; s < ns; ++s) c0[s] = s0[s], nrow[s] = (int)st[s].size(), nv[s] = val_count(s0[s + 1] - s0[s], nrow[s]);
    std::vector<char> absorbed(ns, 0);
    for (int s = 0; s < ns; ++s) {
      const int p = sparent[s];
      if (p < 0 || s0[s + 1] != s0[p] || absorbed[s]) continue;
      if (root_cols && s0[p] >= n - root_cols) continue;  // the root block stays exactly the root columns
      // merged group: columns [c0[s], s0[p+1]), rows = own columns + rows of p beyond its columns
      const long long ncs = s0[s + 1] - c0[s], ncp = s0[p + 1] - s0[p];
      const long long n = ncs + ncp, m = ncs + nrow[p];
      const long long merged = val_count(n, m);
      const long long z = merged - nv[s] - nv[p] + zeros[s] + zeros[p];
      if (n <= amalg_small || (double)z <= amalg_zero_frac * (double)merged) {
        if (n > 96) continue;
        absorbed[s] = 1;
        c0[p] = c0[s];
        nrow[p] = (int)m;
        nv[p] = merged;
        zeros[p] = z;
      }
    }
    // rebuild fundamental arrays with merged groups
    std::vector<int> ns0, keep;
    for (int s = 0; s < ns; ++s)
      if (!absorbed[s]) keep.push_back(s), ns0.push_back(c0[s]);
    const int nn = (int)keep.size();
    ns0.push_back(n);
    std::vector<int> nsn_of(n);
    for (int k = 0; k < nn; ++k)
      for (int c = ns0[k]; c < ns0[k + 1]; ++c) nsn_of[c] = k;
    std::vector<int> nparent(nn, -1);
    for (int k = 0; k < nn; ++k) {
      const int last = ns0[k + 1] - 1;
      if (parent[last] >= 0) nparent[k] = nsn_of[parent[last]];
    }
    std::vector<std::vector<int>> nst(nn), nchild(nn);
    for (int k = 0; k < nn; ++k) {
      const int s = keep[k];
      std::vector<int>& R = nst[k];
      for (int c = ns0[k]; c < ns0[k + 1]; ++c) R.push_back(c);
      const int cend = ns0[k + 1];
      for (int r : st[s])
        if (r >= cend) R.push_back(r);
    }
    for (int k = 0; k < nn; ++k)
      if (nparent[k] >= 0) nchild[nparent[k]].push_back(k);
    s0.swap(ns0), sparent.swap(nparent), st.swap(nst), schild.swap(nchild);
    sn_of.swap(nsn_of);
    ns = nn;
  }
  // ---- multi-level task selection on the supernodal tree ----
  std::vector<long long> w(ns);
  for (int s = 0; s < ns; ++s) {
    const long long nc = s0[s + 1] - s0[s], m = (long long)st[s].size();
    w[s] = nc * m - nc * (nc + 1) / 2 + nc;
  }
  long long wtot = 0;
  for (long long x : w) wtot += x;
  std::vector<char> removed(ns, 0);
  // level 0: subtree roots (one warp per subtree); levels >= 1: chain tasks
  // given by their bottom and top supernodes
  std::vector<std::vector<int>> level_roots, level_tops;
  bool leaf_level = false;
  {
    std::vector<long long> W(ns, 0), Cc(ns, 0), Nsn(ns, 1);
    for (int s = 0; s < ns; ++s) W[s] += w[s], Cc[s] += s0[s + 1] - s0[s];
    for (int s = 0; s < ns; ++s)
      if (sparent[s] >= 0) W[sparent[s]] += W[s], Cc[sparent[s]] += Cc[s], Nsn[sparent[s]] += Nsn[s];
    std::vector<int> picked;
    if (task_cap > 0) {
      std::function<void(int)> pick = [&](int s) {
        const long long ws = Cc[s] + (long long)st[s].size() - (s0[s + 1] - s0[s]);
        if (W[s] <= task_cap && ws <= ws_cap && Nsn[s] <= kMaxTaskSn) {
          picked.push_back(s);
          return;
        }
        for (int ch : schild[s]) pick(ch);
      };
      for (int s = 0; s < ns; ++s)
        if (sparent[s] < 0) pick(s);
    }
    std::function<void(int)> mark_rm = [&](int s) {
      removed[s] = 1;
      for (int ch : schild[s]) mark_rm(ch);
    };
    for (int r : picked) mark_rm(r);
    std::sort(picked.begin(), picked.end());
    if (!picked.empty()) {
      leaf_level = true;
      level_roots.push_back(picked);
      level_tops.push_back(picked);
    }
    // upper part: chains (a supernode with exactly one remaining child joins
    // its child's task), levelled by height; tasks of one level are independent
    std::vector<int> task_of(ns, -1), rem_child(ns, 0), tlevel, tbottom, ttop, tlen;
    for (int s = 0; s < ns; ++s)
      if (!removed[s] && sparent[s] >= 0) rem_child[sparent[s]]++;
    for (int s = 0; s < ns; ++s) {
      if (removed[s]) continue;
      int only = -1;
      if (rem_child[s] == 1)
        for (int ch : schild[s])
          if (!removed[ch]) only = ch;
      if (only >= 0 && tlen[task_of[only]] < kMaxTaskSn) {
        task_of[s] = task_of[only];
        ttop[task_of[s]] = s;
        tlen[task_of[s]]++;
      } else {
        int lv = 0;
        for (int ch : schild[s])
          if (!removed[ch]) lv = std::max(lv, tlevel[task_of[ch]] + 1);
        task_of[s] = (int)tlevel.size();
        tlevel.push_back(lv);
        tbottom.push_back(s);
        ttop.push_back(s);
        tlen.push_back(1);
      }
    }
    int maxlv = -1;
    for (int lv : tlevel) maxlv = std::max(maxlv, lv);
    for (int lv = 0; lv <= maxlv; ++lv) {
      std::vector<int> bots, tops;
      for (std::size_t t = 0; t < tlevel.size(); ++t)
        if (tlevel[t] == lv) bots.push_back(tbottom[t]), tops.push_back(ttop[t]);
      level_roots.push_back(bots);
      level_tops.push_back(tops);
    }
  }
  F.nlevel = (int)level_roots.size();
  // supernode order: tasks level by level, each task a postorder of its
  // (remaining-forest) subtree
  std::vector<int> owner(ns, -1), new_order;
  new_order.reserve(ns);
  std::vector<int> tsn0, tsn1, tlvl;
  std::vector<char> placed(ns, 0);
  std::function<void(int, int)> collect = [&](int s, int t) {
    for (int ch : schild[s])
      if (!placed[ch] && owner[ch] < 0) collect(ch, t);
    owner[s] = t;
    placed[s] = 1;
    new_order.push_back(s);
  };
  F.level_ptr.push_back(0);
  for (int lvl = 0; lvl < F.nlevel; ++lvl) {
    for (std::size_t q = 0; q < level_roots[lvl].size(); ++q) {
      const int t = (int)tsn0.size();
      tsn0.push_back((int)new_order.size());
      if (lvl == 0 && leaf_level) {
        collect(level_roots[lvl][q], t);
      } else {
        // chain bottom .. top (every parent on the way has this chain as its only remaining child)
        int sN = level_roots[lvl][q];
        const int top = level_tops[lvl][q];
        while (true) {
          owner[sN] = t;
          placed[sN] = 1;
          new_order.push_back(sN);
          if (sN == top) break;
          sN = sparent[sN];
        }
      }
      tsn1.push_back((int)new_order.size());
      tlvl.push_back(lvl);
    }
    F.level_ptr.push_back((int)tsn0.size());
  }
  if ((int)new_order.size() != ns) fail(kInternal, "symbolic: task selection did not cover the tree");
  F.ntask = (int)tsn0.size();
  F.top_sn0 = F.nlevel > 0 ? tsn0[F.level_ptr[F.nlevel - 1]] : 0;
  // relabel columns
  std::vector<int> newpos(n);
  {
    int pos = 0;
    for (int s : new_order)
      for (int c = s0[s]; c < s0[s + 1]; ++c) newpos[c] = pos++;
  }
  F.perm.resize(n);
  F.iperm.resize(n);
  for (int k = 0; k < n; ++k) {
    F.perm[newpos[k]] = order[k];
    F.iperm[order[k]] = newpos[k];
  }
  F.nsn = ns;
  F.sn_col0.resize(ns), F.sn_ncol.resize(ns), F.sn_nrow.resize(ns), F.sn_task.resize(ns);
  F.sn_rowoff.resize(ns + 1), F.sn_valoff.resize(ns + 1);
  F.sn_rowoff[0] = F.sn_valoff[0] = 0;
  for (int k = 0; k < ns; ++k) {
    const int s = new_order[k];
    const int nc = s0[s + 1] - s0[s], m = (int)st[s].size();
    F.sn_col0[k] = newpos[s0[s]];
    F.sn_ncol[k] = nc;
    F.sn_nrow[k] = m;
    F.sn_task[k] = owner[s];
    std::vector<int> r;
    r.reserve(m);
    for (int x : st[s]) r.push_back(newpos[x]);
    std::sort(r.begin() + nc, r.end());
    F.rows.insert(F.rows.end(), r.begin(), r.end());
    F.sn_rowoff[k + 1] = F.sn_rowoff[k] + m;
    F.sn_valoff[k + 1] = F.sn_valoff[k] + (long long)nc * m - (long long)nc * (nc + 1) / 2;
    F.flops_factor += (long long)nc * m * m;
  }
  F.nval = F.sn_valoff[ns];
  // task column ranges, contribution rows, slots and fold lists
  F.slot.assign(F.rows.size(), -1);
  F.top_c0 = F.top_sn0 < ns ? F.sn_col0[F.top_sn0] : n;
  F.level_ws.assign(F.nlevel, 0);
  std::vector<std::vector<int>> fold(n);
  for (int t = 0; t < F.ntask; ++t) {
    F.task_sn0.push_back(tsn0[t]);
    F.task_sn1.push_back(tsn1[t]);
    F.task_level.push_back(tlvl[t]);
    const int c0 = F.sn_col0[tsn0[t]];
    const int c1 = F.sn_col0[tsn1[t] - 1] + F.sn_ncol[tsn1[t] - 1];
    F.task_c0.push_back(c0);
    F.task_c1.push_back(c1);
    std::vector<int> cb;
    for (int k = tsn0[t]; k < tsn1[t]; ++k)
      for (long long q = F.sn_rowoff[k]; q < F.sn_rowoff[k + 1]; ++q)
        if (F.rows[q] >= c1) cb.push_back(F.rows[q]);
    std::sort(cb.begin(), cb.end());
    cb.erase(std::unique(cb.begin(), cb.end()), cb.end());
    F.task_cboff.push_back((int)F.cb_rows.size());
    F.task_cblen.push_back((int)cb.size());
    for (std::size_t i = 0; i < cb.size(); ++i) fold[cb[i]].push_back(F.task_cboff[t] + (int)i);
    F.cb_rows.insert(F.cb_rows.end(), cb.begin(), cb.end());
    const int ws = (c1 - c0) + (int)cb.size();
    F.level_ws[tlvl[t]] = std::max(F.level_ws[tlvl[t]], ws);
    if (tlvl[t] == 0) F.max_task_ws = std::max(F.max_task_ws, ws);
    for (int k = tsn0[t]; k < tsn1[t]; ++k)
      for (long long q = F.sn_rowoff[k]; q < F.sn_rowoff[k + 1]; ++q) {
        const int r = F.rows[q];
        if (r < c1) {
          if (r < c0) fail(kInternal, "symbolic: task row below its column range");
          F.slot[q] = r - c0;
        } else {
          F.slot[q] = (c1 - c0) + int(std::lower_bound(cb.begin(), cb.end(), r) - cb.begin());
        }
      }
  }
  // factor values: a task's supernodes are contiguous and every task starts
  // at an even offset (16-byte aligned streams for the bulk copies)
  {
    std::vector<char> tstart(ns, 0);
    long long cover = 0;
    for (int t = 0; t < F.ntask; ++t) tstart[F.task_sn0[t]] = 1, cover += F.task_sn1[t] - F.task_sn0[t];
    if (cover != ns) fail(kInternal, "symbolic: tasks do not partition the supernodes");
    long long v = 0;
    for (int k = 0; k < ns; ++k) {
      if (tstart[k]) v = (v + 1) & ~1LL;
      F.sn_valoff[k] = v;
      v += sn_size(F.sn_ncol[k], F.sn_nrow[k]);
    }
    F.sn_valoff[ns] = v;
    F.nval = (v + 1) & ~1LL;
  }
  // every contribution row must belong to a task of a strictly higher level
  std::vector<int> col_level(n, -1);
  for (int t = 0; t < F.ntask; ++t)
    for (int c = F.task_c0[t]; c < F.task_c1[t]; ++c) col_level[c] = F.task_level[t];
  for (int t = 0; t < F.ntask; ++t)
    for (int i = 0; i < F.task_cblen[t]; ++i)
      if (col_level[F.cb_rows[F.task_cboff[t] + i]] <= F.task_level[t])
        fail(kInternal, "symbolic: contribution row not owned by a higher level");
  F.fold_ptr.assign(n + 1, 0);
  for (int c = 0; c < n; ++c) {
    F.fold_idx.insert(F.fold_idx.end(), fold[c].begin(), fold[c].end());
    F.fold_ptr[c + 1] = (int)F.fold_idx.size();
  }
  return F;
}

/// Host numeric supernodal LDL^T (setup phase) of a matrix with pattern A and
/// values `vals` (natural order, symmetric).  Output: packed strict-lower
/// trapezoids `L` (F.nval) and pivots `D` (F.n), position order.
/// fixed: natural dofs replaced by identity rows/cols (floating subdomains).
inline void factor_host(const SymFactor& F, const Csr& A, const double* vals, const std::vector<int>& fixed,
                        std::vector<double>& L, std::vector<double>& D) {
  const int n = F.n;
  std::vector<char> isfix(n, 0);
  for (int f : fixed) isfix[F.iperm[f]] = 1;
  // full column-major blocks m x ncol per supernode
  std::vector<long long> boff(F.nsn + 1, 0);
  for (int k = 0; k < F.nsn; ++k) boff[k + 1] = boff[k] + (long long)F.sn_nrow[k] * F.sn_ncol[k];
  std::vector<double> blk(boff[F.nsn], 0.0);
  std::vector<int> sn_of(n);
  for (int k = 0; k < F.nsn; ++k)
    for (int c = 0; c < F.sn_ncol[k]; ++c) sn_of[F.sn_col0[k] + c] = k;
  std::vector<int> where(n, -1);
  // scatter lower triangle of P A P^T
  for (int k = 0; k < F.nsn; ++k) {
    const int m = F.sn_nrow[k], nc = F.sn_ncol[k];
    const int* R = &F.rows[F.sn_rowoff[k]];
    for (int i = 0; i < m; ++i) where[R[i]] = i;
    for (int c = 0; c < nc; ++c) {
      const int pc = F.sn_col0[k] + c, nat = F.perm[pc];
      if (isfix[pc]) {
        blk[boff[k] + (long long)c * m + c] = 1.0;
        continue;
      }
      for (int q = A.ptr[nat]; q < A.ptr[nat + 1]; ++q) {
        const int pr = F.iperm[A.col[q]];
        if (pr < pc || isfix[pr]) continue;
        const int i = where[pr];
        if (i < 0) fail(kInternal, "factor_host: entry outside symbolic structure");
        blk[boff[k] + (long long)c * m + i] += vals[q];
      }
    }
    for (int i = 0; i < m; ++i) where[R[i]] = -1;
  }
  D.assign(n, 0.0);
  std::vector<double> W;
  for (int k = 0; k < F.nsn; ++k) {
    const int m = F.sn_nrow[k], nc = F.sn_ncol[k];
    double* B = &blk[boff[k]];
    const int* R = &F.rows[F.sn_rowoff[k]];
    // dense LDL^T of the trapezoid (left-looking inside the supernode)
    for (int j = 0; j < nc; ++j) {
      double* cj = B + (long long)j * m;
      for (int p = 0; p < j; ++p) {
        const double* cp = B + (long long)p * m;
        const double f = cp[j] * D[F.sn_col0[k] + p];
        if (f == 0.0) continue;
        for (int i = j; i < m; ++i) cj[i] -= cp[i] * f;
      }
      const double d = cj[j];
      if (d == 0.0 || !std::isfinite(d)) fail(kSingular, "subdomain saddle factorization failed (zero pivot)");
      D[F.sn_col0[k] + j] = d;
      const double inv = 1.0 / d;
      for (int i = j + 1; i < m; ++i) cj[i] *= inv;
    }
    // update ancestors with W = L_R D L_R^T over off-diagonal rows R
    const int mr = m - nc;
    if (mr == 0) continue;
    W.assign((std::size_t)mr * mr, 0.0);
    for (int p = 0; p < nc; ++p) {
      const double* cp = B + (long long)p * m + nc;
      const double dp = D[F.sn_col0[k] + p];
      for (int b = 0; b < mr; ++b) {
        const double f = cp[b] * dp;
        if (f == 0.0) continue;
        double* wb = &W[(std::size_t)b * mr];
        for (int a = b; a < mr; ++a) wb[a] += cp[a] * f;
      }
    }
    // scatter-subtract into target supernodes
    for (int b = 0; b < mr;) {
      const int t = sn_of[R[nc + b]];
      const int tm = F.sn_nrow[t];
      const int* TR = &F.rows[F.sn_rowoff[t]];
      for (int i = 0; i < tm; ++i) where[TR[i]] = i;
      double* TB = &blk[boff[t]];
      int b2 = b;
      while (b2 < mr && sn_of[R[nc + b2]] == t) {
        const int tc = R[nc + b2] - F.sn_col0[t];
        const double* wb = &W[(std::size_t)b2 * mr];
        double* tcol = TB + (long long)tc * tm;
        for (int a = b2; a < mr; ++a) tcol[where[R[nc + a]]] -= wb[a];
        ++b2;
      }
      for (int i = 0; i < tm; ++i) where[TR[i]] = -1;
      b = b2;
    }
  }
  // pack strict lower trapezoids
  L.assign(F.nval, 0.0);
  for (int k = 0; k < F.nsn; ++k) {
    const int m = F.sn_nrow[k], nc = F.sn_ncol[k];
    long long o = F.sn_valoff[k];
    for (int j = 0; j < nc; ++j)
      for (int i = j + 1; i < m; ++i) L[o++] = blk[boff[k] + (long long)j * m + i];
  }
}

/// Host supernodal solve with the packed layout (validation and the seeded
/// factor check only; the engine's solves run on the device).
inline void solve_host(const SymFactor& F, const std::vector<double>& L, const std::vector<double>& D,
                       double* x_natural) {
  std::vector<double> x(F.n);
  for (int p = 0; p < F.n; ++p) x[p] = x_natural[F.perm[p]];
  for (int k = 0; k < F.nsn; ++k) {
    const int m = F.sn_nrow[k], nc = F.sn_ncol[k];
    const int* R = &F.rows[F.sn_rowoff[k]];
    const double* V = &L[F.sn_valoff[k]];
    for (int j = 0; j < nc; ++j) {
      const double xj = x[R[j]];
      for (int i = j + 1; i < m; ++i) x[R[i]] -= (*V++) * xj;
    }
  }
  for (int p = 0; p < F.n; ++p) x[p] /= D[p];
  for (int k = F.nsn - 1; k >= 0; --k) {
    const int m = F.sn_nrow[k], nc = F.sn_ncol[k];
    const int* R = &F.rows[F.sn_rowoff[k]];
    for (int j = nc - 1; j >= 0; --j) {
      const long long o = F.sn_valoff[k] + (long long)j * (m - 1) - (long long)j * (j - 1) / 2;
      double s = x[R[j]];
      for (int i = j + 1; i < m; ++i) s -= L[o + (i - j - 1)] * x[R[i]];
      x[R[j]] = s;
    }
  }
  for (int p = 0; p < F.n; ++p) x_natural[F.perm[p]] = x[p];
}

/// Host emulation of the device task schedule (warp/CTA tasks level by level,
/// identical slot / contribution / fold semantics) for the CPU validation of
/// the symbolic layout.  x in position order, solved in place.
inline void solve_tasks_host(const SymFactor& F, const std::vector<double>& L, const std::vector<double>& D,
                             std::vector<double>& x) {
  std::vector<double> CB(F.cb_rows.size(), 0.0);
  auto fwd_task = [&](int t, bool also_bwd) {
    const int c0 = F.task_c0[t], c1 = F.task_c1[t], nct = c1 - c0, cbl = F.task_cblen[t];
    std::vector<double> ws(nct + cbl, 0.0);
    for (int i = 0; i < nct; ++i) {
      double v = x[c0 + i];
      for (int q = F.fold_ptr[c0 + i]; q < F.fold_ptr[c0 + i + 1]; ++q) v += CB[F.fold_idx[q]];
      ws[i] = v;
    }
    for (int k = F.task_sn0[t]; k < F.task_sn1[t]; ++k) {
      const int m = F.sn_nrow[k], nc = F.sn_ncol[k];
      const int* sl = &F.slot[F.sn_rowoff[k]];
      const double* V = &L[F.sn_valoff[k]];
      for (int j = 0; j < nc; ++j) {
        const double xj = ws[sl[j]];
        for (int i = j + 1; i < m; ++i) ws[sl[i]] -= (*V++) * xj;
      }
    }
    for (int i = 0; i < nct; ++i) ws[i] /= D[c0 + i];
    for (int i = 0; i < cbl; ++i) CB[F.task_cboff[t] + i] = ws[nct + i];
    if (also_bwd) {
      for (int k = F.task_sn1[t] - 1; k >= F.task_sn0[t]; --k) {
        const int m = F.sn_nrow[k], nc = F.sn_ncol[k];
        const int* sl = &F.slot[F.sn_rowoff[k]];
        for (int j = nc - 1; j >= 0; --j) {
          const long long o = F.sn_valoff[k] + (long long)j * (m - 1) - (long long)j * (j - 1) / 2;
          double s = 0;
          for (int i = j + 1; i < m; ++i) s += L[o + (i - j - 1)] * ws[sl[i]];
          ws[sl[j]] -= s;
        }
      }
    }
    for (int i = 0; i < nct; ++i) x[c0 + i] = ws[i];
  };
  auto bwd_task = [&](int t) {
    const int c0 = F.task_c0[t], c1 = F.task_c1[t], nct = c1 - c0, cbl = F.task_cblen[t];
    std::vector<double> w2(nct + cbl);
    for (int i = 0; i < nct; ++i) w2[i] = x[c0 + i];
    for (int i = 0; i < cbl; ++i) w2[nct + i] = x[F.cb_rows[F.task_cboff[t] + i]];
    for (int k = F.task_sn1[t] - 1; k >= F.task_sn0[t]; --k) {
      const int m = F.sn_nrow[k], nc = F.sn_ncol[k];
      const int* sl = &F.slot[F.sn_rowoff[k]];
      for (int j = nc - 1; j >= 0; --j) {
        const long long o = F.sn_valoff[k] + (long long)j * (m - 1) - (long long)j * (j - 1) / 2;
        double s = 0;
        for (int i = j + 1; i < m; ++i) s += L[o + (i - j - 1)] * w2[sl[i]];
        w2[sl[j]] -= s;
      }
    }
    for (int i = 0; i < nct; ++i) x[c0 + i] = w2[i];
  };
  for (int l = 0; l < F.nlevel; ++l)
    for (int t = F.level_ptr[l]; t < F.level_ptr[l + 1]; ++t) fwd_task(t, l == F.nlevel - 1);
  for (int l = F.nlevel - 2; l >= 0; --l)
    for (int t = F.level_ptr[l]; t < F.level_ptr[l + 1]; ++t) bwd_task(t);
}

}  // namespace pf

namespace pf {

/// Structure for the multifrontal numeric factorisation on the device: the
/// supernodal tree in final numbering, fronts (m x m column-major) per
/// supernode, children lists with relative row positions for the
/// extend-add, and supernodes grouped by height (all supernodes of one height
/// are independent).
struct FrontMaps {
  std::vector<int> parent, height;
  int nheight = 0;
  std::vector<int> height_ptr, height_sn;  // supernodes by height
  std::vector<long long> foff;             // front offset per supernode (doubles)
  long long fsize = 0;
  std::vector<int> ch_ptr, ch_idx;         // children (ascending)
  std::vector<long long> rp_off;           // per supernode as a child: relpos offset
  std::vector<int> relpos;                 // rows beyond own columns -> index in parent rows
};

inline FrontMaps build_front_maps(const SymFactor& F) {
  FrontMaps M;
  const int ns = F.nsn;
  std::vector<int> sn_of(F.n);
  for (int k = 0; k < ns; ++k)
    for (int c = 0; c < F.sn_ncol[k]; ++c) sn_of[F.sn_col0[k] + c] = k;
  M.parent.assign(ns, -1);
  for (int k = 0; k < ns; ++k)
    if (F.sn_nrow[k] > F.sn_ncol[k]) M.parent[k] = sn_of[F.rows[F.sn_rowoff[k] + F.sn_ncol[k]]];
  M.height.assign(ns, 0);
  std::vector<int> order(ns);
  std::iota(order.begin(), order.end(), 0);
  // children precede parents in the final numbering
  for (int k = 0; k < ns; ++k)
    if (M.parent[k] >= 0) {
      if (M.parent[k] <= k) fail(kInternal, "front maps: parent not after child");
      M.height[M.parent[k]] = std::max(M.height[M.parent[k]], M.height[k] + 1);
    }
  for (int h : M.height) M.nheight = std::max(M.nheight, h + 1);
  M.height_ptr.assign(M.nheight + 1, 0);
  for (int h : M.height) M.height_ptr[h + 1]++;
  for (int h = 0; h < M.nheight; ++h) M.height_ptr[h + 1] += M.height_ptr[h];
  M.height_sn.resize(ns);
  {
    std::vector<int> pos(M.height_ptr.begin(), M.height_ptr.end() - 1);
    for (int k = 0; k < ns; ++k) M.height_sn[pos[M.height[k]]++] = k;
  }
  M.foff.resize(ns + 1);
  M.foff[0] = 0;
  for (int k = 0; k < ns; ++k) M.foff[k + 1] = M.foff[k] + (long long)F.sn_nrow[k] * F.sn_nrow[k];
  M.fsize = M.foff[ns];
  std::vector<std::vector<int>> ch(ns);
  for (int k = 0; k < ns; ++k)
    if (M.parent[k] >= 0) ch[M.parent[k]].push_back(k);
  M.ch_ptr.assign(ns + 1, 0);
  for (int k = 0; k < ns; ++k) {
    M.ch_idx.insert(M.ch_idx.end(), ch[k].begin(), ch[k].end());
    M.ch_ptr[k + 1] = (int)M.ch_idx.size();
  }
  M.rp_off.assign(ns + 1, 0);
  for (int k = 0; k < ns; ++k) {
    const int p = M.parent[k];
    const int nc = F.sn_ncol[k], m = F.sn_nrow[k];
    if (p >= 0) {
      const int* pr = &F.rows[F.sn_rowoff[p]];
      const int pm = F.sn_nrow[p];
      for (int i = nc; i < m; ++i) {
        const int r = F.rows[F.sn_rowoff[k] + i];
        const int* it = std::lower_bound(pr, pr + pm, r);
        if (it == pr + pm || *it != r) fail(kInternal, "front maps: child row not in parent structure");
        M.relpos.push_back(int(it - pr));
      }
    }
    M.rp_off[k + 1] = (long long)M.relpos.size();
  }
  return M;
}

/// Where the lower-triangle entries of A go in the fronts: for supernode k,
/// entries [as_ptr[k], as_ptr[k+1]) with value index (into the subdomain's K
/// values; -1 = unit diagonal of a fixed dof) and front position.
struct AScatter {
  std::vector<int> ptr, kidx, fpos;
};

/// A given by its pattern (natural numbering) and, per entry, the index of its
/// value in the subdomain's K value array (kmap, nullptr = identity).
inline AScatter build_ascatter(const SymFactor& F, const FrontMaps& M, const Csr& A, const int* kmap,
                               const std::vector<int>& fixed_natural) {
  const int n = F.n;
  std::vector<char> isfix(n, 0);
  for (int f : fixed_natural) isfix[F.iperm[f]] = 1;
  std::vector<int> sn_of(n);
  for (int k = 0; k < F.nsn; ++k)
    for (int c = 0; c < F.sn_ncol[k]; ++c) sn_of[F.sn_col0[k] + c] = k;
  std::vector<std::vector<std::pair<int, int>>> per(F.nsn);
  std::vector<int> where(n, -1);
  for (int k = 0; k < F.nsn; ++k) {
    const int m = F.sn_nrow[k];
    const int* R = &F.rows[F.sn_rowoff[k]];
    for (int i = 0; i < m; ++i) where[R[i]] = i;
    for (int c = 0; c < F.sn_ncol[k]; ++c) {
      const int pc = F.sn_col0[k] + c, nat = F.perm[pc];
      if (isfix[pc]) {
        per[k].emplace_back(-1, c + c * m);
        continue;
      }
      for (int q = A.ptr[nat]; q < A.ptr[nat + 1]; ++q) {
        const int pr = F.iperm[A.col[q]];
        if (pr < pc || isfix[pr]) continue;
        const int i = where[pr];
        if (i < 0) fail(kInternal, "ascatter: entry outside the symbolic structure");
        per[k].emplace_back(kmap ? kmap[q] : q, i + c * m);
      }
    }
    for (int i = 0; i < m; ++i) where[R[i]] = -1;
  }
  (void)M;
  AScatter S;
  S.ptr.assign(F.nsn + 1, 0);
  for (int k = 0; k < F.nsn; ++k) {
    for (auto& e : per[k]) S.kidx.push_back(e.first), S.fpos.push_back(e.second);
    S.ptr[k + 1] = (int)S.kidx.size();
  }
  return S;
}

/// Convert factor values from the packed column-major trapezoid (factor_host)
/// to the panel-blocked sweep layout (pf_layout.hpp), in place; each panel's
/// triangle unit receives the inverse of its unit-lower diagonal block.
inline void to_blocked(const SymFactor& F, std::vector<double>& L) {
  std::vector<double> out(L.size(), 0.0);
  std::vector<double> T, X;
  for (int k = 0; k < F.nsn; ++k) {
    const int nc = F.sn_ncol[k], m = F.sn_nrow[k];
    const long long o = F.sn_valoff[k];
    auto packed = [&](int i, int j) { return L[o + (long long)j * (m - 1) - (long long)j * (j - 1) / 2 + (i - j - 1)]; };
    for (int j = 0; j < nc; ++j)
      for (int i = j + 1; i < m; ++i) out[o + blk_off(nc, m, i, j)] = packed(i, j);
    for (int p0 = 0; p0 < nc; p0 += kPW) {
      const int pw = std::min(kPW, nc - p0);
      X.assign((std::size_t)pw * pw, 0.0);  // X = Linv, column-major
      for (int j = 0; j < pw; ++j) {
        X[j + j * pw] = 1.0;
        for (int i = j + 1; i < pw; ++i) {
          double acc = 0.0;
          for (int q = j; q < i; ++q) acc += packed(p0 + i, p0 + q) * X[q + j * pw];
          X[i + j * pw] = -acc;
        }
      }
      for (int j = 0; j < pw; ++j)
        for (int i = j + 1; i < pw; ++i) out[o + blk_off(nc, m, p0 + i, p0 + j)] = X[i + j * pw];
    }
  }
  L.swap(out);
}

}  // namespace pf
