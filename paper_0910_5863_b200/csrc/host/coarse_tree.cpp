// Nested-dissection tree over the primal unknowns (see coarse_tree.hpp).
#include "coarse_tree.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace b200 {
namespace {

constexpr int kT = 64;
int rup(int x) { return (x + kT - 1) / kT * kT; }

struct Box {
  int lo[3], hi[3];
  int parent = -1;
  std::vector<int> kids;
};

// boxes[d] = the boxes of depth d; false when a box cannot be split
bool build_boxes(const int lattice[3], int depth, std::vector<std::vector<Box>>& boxes) {
  boxes.assign(depth + 1, {});
  Box root;
  for (int a = 0; a < 3; ++a) {
    root.lo[a] = 0;
    root.hi[a] = lattice[a];
  }
  boxes[0].push_back(root);
  for (int d = 1; d <= depth; ++d) {
    for (int b = 0; b < static_cast<int>(boxes[d - 1].size()); ++b) {
      const Box par = boxes[d - 1][b];
      int cuts[3][3], nparts[3];
      bool any = false;
      for (int a = 0; a < 3; ++a) {
        const int ext = par.hi[a] - par.lo[a];
        if (ext >= 2) {
          nparts[a] = 2;
          cuts[a][0] = par.lo[a];
          cuts[a][1] = par.lo[a] + (ext + 1) / 2;  // the block partition's cut (shard.py partition) for two parts
          cuts[a][2] = par.hi[a];
          any = true;
        } else {
          nparts[a] = 1;
          cuts[a][0] = par.lo[a];
          cuts[a][1] = par.hi[a];
        }
      }
      if (!any) return false;
      for (int z = 0; z < nparts[2]; ++z)
        for (int y = 0; y < nparts[1]; ++y)
          for (int x = 0; x < nparts[0]; ++x) {
            Box c;
            const int ix[3] = {x, y, z};
            for (int a = 0; a < 3; ++a) {
              c.lo[a] = cuts[a][ix[a]];
              c.hi[a] = cuts[a][ix[a] + 1];
            }
            c.parent = b;
            boxes[d - 1][b].kids.push_back(static_cast<int>(boxes[d].size()));
            boxes[d].push_back(c);
          }
    }
  }
  return true;
}

bool inside(const Box& b, const int lo[3], const int hi[3]) {
  for (int a = 0; a < 3; ++a)
    if (lo[a] < b.lo[a] || hi[a] > b.hi[a]) return false;
  return true;
}

// gather CSR from (position, child, cidx, src) tuples produced in child order
void to_csr(std::size_t npos, const std::vector<long long>& pos, const std::vector<int>& ch,
            const std::vector<int>& ci, const std::vector<long long>& sr, std::vector<int>& ptr,
            std::vector<int>& child, std::vector<int>& cidx, std::vector<long long>& src) {
  ptr.assign(npos + 1, 0);
  for (long long p : pos) ++ptr[p + 1];
  for (std::size_t i = 0; i < npos; ++i) ptr[i + 1] += ptr[i];
  std::vector<int> fill(ptr.begin(), ptr.end() - 1);
  child.resize(pos.size());
  cidx.resize(pos.size());
  src.resize(pos.size());
  for (std::size_t e = 0; e < pos.size(); ++e) {
    const int at = fill[pos[e]]++;
    child[at] = ch[e];
    cidx[at] = ci[e];
    src[at] = sr[e];
  }
}

}  // namespace

int coarse_tree_max_depth(const int lattice[3]) {
  int d = 0;
  std::vector<std::vector<Box>> boxes;
  while (d < 6 && build_boxes(lattice, d + 1, boxes)) ++d;
  return d;
}

int coarse_tree_shard_depth(const int lattice[3], const std::vector<int>& owner, int max_depth) {
  // deeper boxes nest inside the depth-1 boxes, so those decide
  if (max_depth < 1) return 0;
  std::vector<std::vector<Box>> boxes;
  if (!build_boxes(lattice, 1, boxes)) return 0;
  for (const Box& b : boxes[1]) {
    int r = -1;
    for (int z = b.lo[2]; z < b.hi[2]; ++z)
      for (int y = b.lo[1]; y < b.hi[1]; ++y)
        for (int x = b.lo[0]; x < b.hi[0]; ++x) {
          const int o = owner[(static_cast<std::size_t>(z) * lattice[1] + y) * lattice[0] + x];
          if (r < 0) r = o;
          if (o != r) return 0;
        }
  }
  return max_depth;
}

CoarseTree plan_coarse_tree(const std::vector<CoarseLeaf>& leaves, const int lattice[3], int n_primal, int depth,
                            int root_inverse_max, bool symbolic, const CoarseBounds* bounds) {
  CoarseTree t;
  t.depth = depth;
  std::vector<std::vector<Box>> boxes;
  if (!build_boxes(lattice, depth, boxes)) throw std::invalid_argument("coarse tree: depth too large for the lattice");
  const int nl = static_cast<int>(leaves.size());
  // bounding box of each primal unknown's substructures
  std::vector<int> lo, hi;
  if (bounds) {  // sharded: the bounds over every rank's substructures
    if (bounds->lo.size() != 3 * (size_t)n_primal || bounds->hi.size() != 3 * (size_t)n_primal)
      throw std::invalid_argument("coarse tree: bounds do not match the primal unknowns");
    lo = bounds->lo;
    hi = bounds->hi;
  } else {
    lo.assign(3 * (size_t)n_primal, 1 << 30);
    hi.assign(3 * (size_t)n_primal, -1);
    for (const CoarseLeaf& l : leaves)
      for (int k : l.coarse)
        for (int a = 0; a < 3; ++a) {
          lo[3 * (size_t)k + a] = std::min(lo[3 * (size_t)k + a], l.coord[a]);
          hi[3 * (size_t)k + a] = std::max(hi[3 * (size_t)k + a], l.coord[a] + 1);
        }
  }
  // owner box of each unknown: the deepest box containing its bounding box
  std::vector<std::vector<std::vector<int>>> own(depth + 1);
  for (int d = 0; d <= depth; ++d) own[d].resize(boxes[d].size());
  for (int k = 0; k < n_primal; ++k) {
    int d = 0, b = 0;
    if (hi[3 * (size_t)k] < 0) {  // no leaf here holds it (sharded: another rank's): the top
      own[0][0].push_back(k);
      continue;
    }
    while (d < depth) {
      int next = -1;
      for (int c : boxes[d][b].kids)
        if (inside(boxes[d + 1][c], &lo[3 * (size_t)k], &hi[3 * (size_t)k])) {
          next = c;
          break;
        }
      if (next < 0) break;
      ++d;
      b = next;
    }
    own[d][b].push_back(k);  // ascending: k increases
  }
  // bottom box of each leaf
  std::vector<int> leaf_box(nl);
  for (int i = 0; i < nl; ++i) {
    int b = 0;
    for (int d = 0; d < depth; ++d) {
      int next = -1;
      const int c0[3] = {leaves[i].coord[0], leaves[i].coord[1], leaves[i].coord[2]};
      const int c1[3] = {c0[0] + 1, c0[1] + 1, c0[2] + 1};
      for (int c : boxes[d][b].kids)
        if (inside(boxes[d + 1][c], c0, c1)) {
          next = c;
          break;
        }
      if (next < 0) throw std::logic_error("coarse tree: leaf outside the lattice");
      b = next;
    }
    leaf_box[i] = b;
  }
  // fronts exist for the boxes that hold one of these leaves (all of them on
  // one GPU; a rank's own boxes when sharded): local index per box
  std::vector<std::vector<int>> local(depth + 1);
  for (int d = 0; d <= depth; ++d) local[d].assign(boxes[d].size(), -1);
  for (int i = 0; i < nl; ++i) local[depth][leaf_box[i]] = 0;
  for (int d = depth; d >= 1; --d)
    for (int b = 0; b < static_cast<int>(boxes[d].size()); ++b)
      if (local[d][b] >= 0) local[d - 1][boxes[d][b].parent] = 0;
  for (int d = 0; d <= depth; ++d) {
    int n = 0;
    for (int& v : local[d])
      if (v >= 0) v = n++;
  }
  // update sets, bottom-up
  std::vector<int> mark(n_primal, -1);
  int stamp = 0;
  std::vector<std::vector<std::vector<int>>> upd(depth + 1);
  for (int d = depth; d >= 0; --d) {
    upd[d].resize(boxes[d].size());
    std::vector<std::vector<int>> lists(boxes[d].size());
    if (d == depth) {
      for (int i = 0; i < nl; ++i)
        for (int k : leaves[i].coarse) lists[leaf_box[i]].push_back(k);
    } else {
      for (int b = 0; b < static_cast<int>(boxes[d].size()); ++b)
        for (int c : boxes[d][b].kids) lists[b].insert(lists[b].end(), upd[d + 1][c].begin(), upd[d + 1][c].end());
    }
    for (int b = 0; b < static_cast<int>(boxes[d].size()); ++b) {
      ++stamp;
      for (int k : own[d][b]) mark[k] = stamp;
      std::vector<int>& u = upd[d][b];
      for (int k : lists[b])
        if (mark[k] != stamp) {
          mark[k] = stamp;
          u.push_back(k);
        }
      std::sort(u.begin(), u.end());
    }
  }
  if (!upd[0][0].empty()) throw std::logic_error("coarse tree: the top front passes unknowns up");
  t.top = own[0][0];
  // fronts of depth d >= 1: level index depth - d
  t.levels.resize(depth);
  for (int d = depth; d >= 1; --d) {
    CoarseTree::Level& L = t.levels[depth - d];
    long long fv = 0, ao = 0, dof = 0, co = 0;
    for (int b = 0; b < static_cast<int>(boxes[d].size()); ++b) {
      if (local[d][b] < 0) continue;
      L.fronts.emplace_back();
      CoarseTree::Front& f = L.fronts.back();
      f.parent = d > 1 ? local[d - 1][boxes[d][b].parent] : -1;
      f.own = own[d][b];
      f.upd = upd[d][b];
      f.PE = rup(std::max<int>(static_cast<int>(f.own.size()), 1));
      f.NF = f.PE + rup(std::max<int>(static_cast<int>(f.upd.size()), 1));
      f.fv_off = fv;
      f.a_off = ao;
      f.d_off = dof;
      f.cmap_off = co;
      fv += f.NF;
      ao += (long long)f.NF * f.NF;
      dof += (long long)(f.PE / kT) * kT * kT;
      co += f.NF - f.PE;
      L.max_NF = std::max(L.max_NF, f.NF);
      L.max_PE = std::max(L.max_PE, f.PE);
      L.max_M = std::max(L.max_M, f.NF - f.PE);
      const double e = static_cast<double>(f.own.size()), c = static_cast<double>(f.upd.size());
      t.flops += e * e * e / 3.0 + e * e * c + e * c * c;
      t.apply_bytes += 2.0 * (e * (e + 1) / 2 + e * c) * 8.0;
    }
    L.arena = fv;
    L.a_size = ao;
    L.d_size = dof;
    L.cmap.assign(co, -1);
  }
  {
    const double n = static_cast<double>(t.top.size());
    const bool inv = rup(std::max<int>(static_cast<int>(t.top.size()), 1)) <= root_inverse_max;
    t.flops += inv ? n * n * n : n * n * n / 3.0;
    t.apply_bytes += n * n * 8.0;
  }
  if (depth > 0)
    for (int& b : leaf_box) b = local[depth][b];
  t.leaf_box = std::move(leaf_box);
  t.n_primal = n_primal;
  if (!symbolic) complete_coarse_tree(t, leaves);
  return t;
}

void complete_coarse_tree(CoarseTree& t, const std::vector<CoarseLeaf>& leaves) {
  const int depth = t.depth, nl = static_cast<int>(leaves.size()), n_primal = t.n_primal;
  const std::vector<int>& leaf_box = t.leaf_box;
  // forward gathers and backward maps, parent by parent: the parent's rows are
  // stamped into a direct map, then its children are visited in ascending
  // order, so every position's entry list is ascending by child
  std::vector<int> rowmap(n_primal, -1), rstamp(n_primal, -1);
  int pstamp = 0;
  auto stamp_front = [&](const CoarseTree::Front& f) {
    ++pstamp;
    for (std::size_t i = 0; i < f.own.size(); ++i) {
      rowmap[f.own[i]] = static_cast<int>(i);
      rstamp[f.own[i]] = pstamp;
    }
    for (std::size_t i = 0; i < f.upd.size(); ++i) {
      rowmap[f.upd[i]] = f.PE + static_cast<int>(i);
      rstamp[f.upd[i]] = pstamp;
    }
  };
  auto stamp_top = [&]() {
    ++pstamp;
    for (std::size_t i = 0; i < t.top.size(); ++i) {
      rowmap[t.top[i]] = static_cast<int>(i);
      rstamp[t.top[i]] = pstamp;
    }
  };
  auto row = [&](int k) {
    if (rstamp[k] != pstamp) throw std::logic_error("coarse tree: unknown missing from its parent front");
    return rowmap[k];
  };
  t.leaf_cmap.resize(nl);
  {
    std::vector<long long> pos, sr;
    std::vector<int> ch, ci;
    pos.reserve(nl * 64);
    sr.reserve(nl * 64);
    ch.reserve(nl * 64);
    ci.reserve(nl * 64);
    const int nparent = depth == 0 ? 1 : static_cast<int>(t.levels[0].fronts.size());
    std::vector<std::vector<int>> kids(nparent);
    for (int i = 0; i < nl; ++i) kids[depth == 0 ? 0 : leaf_box[i]].push_back(i);
    for (int pf = 0; pf < nparent; ++pf) {
      long long base = 0;
      if (depth == 0) {
        stamp_top();
      } else {
        stamp_front(t.levels[0].fronts[pf]);
        base = t.levels[0].fronts[pf].fv_off;
      }
      for (int i : kids[pf]) {
        const auto& cs = leaves[i].coarse;
        t.leaf_cmap[i].resize(cs.size());
        for (std::size_t c = 0; c < cs.size(); ++c) {
          const long long p = base + row(cs[c]);
          t.leaf_cmap[i][c] = static_cast<int>(p);
          pos.push_back(p);
          ch.push_back(i);
          ci.push_back(static_cast<int>(c));
          sr.push_back(leaves[i].src0 + static_cast<long long>(c));
        }
      }
    }
    if (depth == 0)
      to_csr(t.top.size(), pos, ch, ci, sr, t.top_ptr, t.top_child, t.top_cidx, t.top_src);
    else
      to_csr(t.levels[0].arena, pos, ch, ci, sr, t.levels[0].ptr, t.levels[0].child, t.levels[0].cidx,
             t.levels[0].src);
  }
  for (int l = 0; l < depth; ++l) {  // children: levels[l]; parents: levels[l + 1] or the top
    CoarseTree::Level& C = t.levels[l];
    const bool to_top = l + 1 == depth;
    std::vector<long long> pos, sr;
    std::vector<int> ch, ci;
    const int nparent = to_top ? 1 : static_cast<int>(t.levels[l + 1].fronts.size());
    std::vector<std::vector<int>> kids(nparent);
    for (int fi = 0; fi < static_cast<int>(C.fronts.size()); ++fi) kids[to_top ? 0 : C.fronts[fi].parent].push_back(fi);
    for (int pf = 0; pf < nparent; ++pf) {
      long long base = 0;
      if (to_top) {
        stamp_top();
      } else {
        stamp_front(t.levels[l + 1].fronts[pf]);
        base = t.levels[l + 1].fronts[pf].fv_off;
      }
      for (int fi : kids[pf]) {
        const CoarseTree::Front& f = C.fronts[fi];
        for (std::size_t c = 0; c < f.upd.size(); ++c) {
          const long long p = base + row(f.upd[c]);
          C.cmap[f.cmap_off + c] = static_cast<int>(p);
          pos.push_back(p);
          ch.push_back(fi);
          ci.push_back(static_cast<int>(c));
          sr.push_back(f.fv_off + f.PE + static_cast<long long>(c));
        }
      }
    }
    if (to_top)
      to_csr(t.top.size(), pos, ch, ci, sr, t.top_ptr, t.top_child, t.top_cidx, t.top_src);
    else
      to_csr(t.levels[l + 1].arena, pos, ch, ci, sr, t.levels[l + 1].ptr, t.levels[l + 1].child,
             t.levels[l + 1].cidx, t.levels[l + 1].src);
  }
}

double coarse_tree_cost(const CoarseTree& t, int applies, int root_inverse_max) {
  // rates measured on the B200 (round-2 depth sweeps on cfg3/cfg4):
  // batched DMMA factorization, the batched front sweeps, the dense root
  // sweeps; the dataflow Cholesky's pivot chain per 64-column step (~13 us,
  // the levels run one after the other) and the latency of a level per apply
  // (gather + two sweeps or two explicit GEMVs)
  for (const auto& L : t.levels)
    if (L.max_NF > 24576) return 1e30;  // the batched sweeps keep a front's vector in shared memory
  const double n = static_cast<double>(t.top.size());
  const bool inv = rup(std::max<int>(static_cast<int>(t.top.size()), 1)) <= root_inverse_max;
  double steps = std::ceil(n / kT) * (inv ? 2 : 1);
  for (const auto& L : t.levels) steps += L.max_PE / kT;
  // per level: host planning and index uploads, the assemble / pad / copy
  // launches and the start-up of one more batched factorization (measured
  // 0.3-0.7 ms per extra level on cfg3/cfg4)
  const double setup = t.flops / 20e12 + steps * 13e-6 + 0.4e-3 * static_cast<double>(t.levels.size());
  const double top_bytes = n * n * 8.0;
  // a level's two sweeps are a chain of 64-row block steps over few fronts:
  // measured 26-35 us per level and apply on cfg3/cfg4 (3 to 7 block steps)
  double level_latency = 0;
  for (const auto& L : t.levels) level_latency += 12e-6 + 6e-6 * (L.max_PE / kT);
  const double per_apply =
      (t.apply_bytes - top_bytes) / 3e12 + top_bytes / (inv ? 4e12 : 0.8e12) + level_latency;
  return setup + applies * per_apply;
}

}  // namespace b200
