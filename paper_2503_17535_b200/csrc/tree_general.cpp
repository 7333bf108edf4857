// tree_general.cpp -- host planning of HPS on general (adaptive) trees; see tree_general.hpp.
#include "tree_general.hpp"

#include <algorithm>
#include <functional>
#include <cmath>
#include <map>
#include <set>
#include <exception>
#include <stdexcept>
#include <thread>

namespace hpsg {

namespace {
const int kOff[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}, {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

HostMat mm(const HostMat& a, const HostMat& b) {
  HostMat c(a.r, b.c);
  for (int j = 0; j < b.c; ++j)
    for (int l = 0; l < a.c; ++l) {
      const double v = b(l, j);
      if (v == 0.0) continue;
      for (int i = 0; i < a.r; ++i) c(i, j) += a(i, l) * v;
    }
  return c;
}
HostMat identity(int n) {
  HostMat m(n, n);
  for (int i = 0; i < n; ++i) m(i, i) = 1.0;
  return m;
}
}  // namespace

// ---------------------------------------------------------------- layouts (proj/src/layout.cpp:10-83)
int Layout::npts() const {
  if (!split) return panel_pts();
  int n = 0;
  for (const auto& s : sub) n += s.npts();
  return n;
}
int Layout::max_level() const {
  if (!split) return 0;
  int m = 0;
  for (const auto& s : sub) m = std::max(m, s.max_level());
  return m + 1;
}
bool Layout::operator==(const Layout& o) const {
  if (split != o.split || q != o.q || fdim != o.fdim) return false;
  if (!split) return true;
  for (size_t i = 0; i < sub.size(); ++i)
    if (sub[i] != o.sub[i]) return false;
  return true;
}
std::string Layout::key() const {
  if (!split) return "p";
  std::string s = "(";
  for (const auto& k : sub) s += k.key();
  return s + ")";
}
Layout Layout::panel(int q, int fdim) {
  Layout l;
  l.q = q;
  l.fdim = fdim;
  return l;
}
Layout Layout::split_of(std::vector<Layout> kids) {
  if (kids.empty()) throw std::runtime_error("PanelLayout::split_of: empty");
  Layout l;
  l.q = kids[0].q;
  l.fdim = kids[0].fdim;
  l.split = true;
  l.sub = std::move(kids);
  return l;
}
Layout layout_meet(const Layout& a, const Layout& b) {
  if (!a.split || !b.split) return a.split ? b : a;  // the coarser of the two
  std::vector<Layout> kids;
  for (size_t i = 0; i < a.sub.size(); ++i) kids.push_back(layout_meet(a.sub[i], b.sub[i]));
  return Layout::split_of(std::move(kids));
}

FaceProjection face_projection(int q) {
  // proj/src/spectral.cpp:454-483: Gauss panel <-> its four quadrant panels, tensor barycentric rules
  std::vector<double> x, w;
  gauss_rule(q, x, w);
  std::vector<double> lo(q), hi(q);
  for (int i = 0; i < q; ++i) lo[i] = (x[i] - 1.0) / 2.0, hi[i] = (x[i] + 1.0) / 2.0;
  const HostMat r1[2] = {bary_interp(x, lo), bary_interp(x, hi)};
  const int qq = q * q;
  FaceProjection fp;
  fp.refine = HostMat(4 * qq, qq);
  for (int hu = 0; hu < 2; ++hu)
    for (int hv = 0; hv < 2; ++hv)
      for (int a = 0; a < q; ++a)
        for (int b = 0; b < q; ++b)
          for (int c = 0; c < q; ++c)
            for (int d = 0; d < q; ++d)
              fp.refine((hu * 2 + hv) * qq + a * q + b, c * q + d) = r1[hu](a, c) * r1[hv](b, d);
  fp.coarsen = HostMat(qq, 4 * qq);
  for (int iu = 0; iu < q; ++iu)
    for (int iv = 0; iv < q; ++iv) {
      const int hu = x[iu] > 0.0 ? 1 : 0, hv = x[iv] > 0.0 ? 1 : 0;
      const HostMat ru = bary_interp(hu ? hi : lo, {x[iu]});
      const HostMat rv = bary_interp(hv ? hi : lo, {x[iv]});
      for (int a = 0; a < q; ++a)
        for (int b = 0; b < q; ++b) fp.coarsen(iu * q + iv, (hu * 2 + hv) * qq + a * q + b) = ru(0, a) * rv(0, b);
    }
  return fp;
}

namespace {
HostMat blockdiag_transfer(const Layout& from, const Layout& to, const FaceProjection& proj) {
  HostMat out(to.npts(), from.npts());
  int ro = 0, co = 0;
  for (size_t i = 0; i < from.sub.size(); ++i) {
    const HostMat b = layout_transfer(from.sub[i], to.sub[i], proj);
    for (int j = 0; j < b.c; ++j)
      for (int r = 0; r < b.r; ++r) out(ro + r, co + j) = b(r, j);
    ro += b.r;
    co += b.c;
  }
  return out;
}
}  // namespace

HostMat layout_transfer(const Layout& from, const Layout& to, const FaceProjection& proj) {
  if (from.fdim != 2) throw std::runtime_error("layout_transfer: only face (2D-panel) transfers are needed");
  if (!from.split && !to.split) return identity(from.panel_pts());
  if (from.split && to.split) return blockdiag_transfer(from, to, proj);
  if (!from.split) {  // refine one level, then recurse into the sub-layouts
    const Layout one = Layout::split_of(std::vector<Layout>(4, Layout::panel(from.q, 2)));
    return mm(blockdiag_transfer(one, to, proj), proj.refine);
  }
  const Layout one = Layout::split_of(std::vector<Layout>(4, Layout::panel(to.q, 2)));
  return mm(proj.coarsen, blockdiag_transfer(from, one, proj));
}

// ---------------------------------------------------------------- tree
void finalize_gtree(GTree& t) {
  const int n = int(t.depth.size());
  if (t.dim != 2 && t.dim != 3) throw std::runtime_error("hpsg_create_tree: dim must be 2 or 3");
  if (n < 1) throw std::runtime_error("hpsg_create_tree: empty tree");
  t.q = t.p - 2;
  t.nchild = t.dim == 2 ? 4 : 8;
  t.nface = 2 * t.dim;
  t.parent.assign(n, -1);
  for (int i = 0; i < n; ++i) {
    if (t.nch[i] != 0 && t.nch[i] != t.nchild)
      throw std::runtime_error(fmt("hpsg_create_tree: node %d has %d children (0 or %d)", i, t.nch[i], t.nchild));
    for (int c = 0; c < t.nch[i]; ++c) {
      const int k = t.child[i][c];
      if (k <= 0 || k >= n || t.parent[k] >= 0) throw std::runtime_error(fmt("hpsg_create_tree: bad child of node %d", i));
      t.parent[k] = i;
      if (t.depth[k] != t.depth[i] + 1) throw std::runtime_error(fmt("hpsg_create_tree: depth of node %d", k));
      for (int a = 0; a < 3; ++a) {  // the child box is the kOff[c] sub-box of the parent (mesh.cpp:27-52)
        const double mid = 0.5 * (t.lo[3 * i + a] + t.hi[3 * i + a]);
        const double elo = (a < t.dim && kOff[c][a]) ? mid : t.lo[3 * i + a];
        const double ehi = (a < t.dim && !kOff[c][a]) ? mid : t.hi[3 * i + a];
        if (a < t.dim && (t.lo[3 * k + a] != elo || t.hi[3 * k + a] != ehi))
          throw std::runtime_error(fmt("hpsg_create_tree: node %d is not child slot %d of node %d", k, c, i));
      }
    }
  }
  if (t.depth[0] != 0) throw std::runtime_error("hpsg_create_tree: node 0 must be the root");
  for (int i = 1; i < n; ++i)
    if (t.parent[i] < 0) throw std::runtime_error(fmt("hpsg_create_tree: node %d is unreachable", i));
  // depth-first levels and leaves (DiscretizationTree::finalize, mesh.cpp:54-71)
  t.levels.clear();
  std::vector<int> dfs_leaves;
  std::vector<int> stack{0};
  while (!stack.empty()) {
    const int id = stack.back();
    stack.pop_back();
    if ((int)t.levels.size() <= t.depth[id]) t.levels.resize(t.depth[id] + 1);
    t.levels[t.depth[id]].push_back(id);
    if (t.nch[id] == 0)
      dfs_leaves.push_back(id);
    else
      for (int c = t.nchild - 1; c >= 0; --c) stack.push_back(t.child[id][c]);
  }
  if (!t.leaves.empty() && t.leaves != dfs_leaves)
    throw std::runtime_error("hpsg_create_tree: leaves are not in depth-first order");
  t.leaves = dfs_leaves;
  t.leaf_ord.assign(n, -1);
  for (size_t i = 0; i < t.leaves.size(); ++i) t.leaf_ord[t.leaves[i]] = int(i);
}

// ---------------------------------------------------------------- plan
GeneralPlan make_general_plan(GTree tree, bool implicit_root) {
  finalize_gtree(tree);
  GeneralPlan g;
  g.tree = std::move(tree);
  const GTree& t = g.tree;
  const int n = int(t.depth.size()), dim = t.dim, nf = t.nface, nc = t.nchild, q = t.q;
  const auto& ifs = ifaces(dim);
  const int nquad = dim == 2 ? 2 : 4;
  if (nc == 4 && t.nch[0] == 0) throw std::runtime_error("hpsg_create_tree: a single-leaf tree has no merge");
  if (t.nch[0] == 0) throw std::runtime_error("hpsg_create_tree: a single-leaf tree has no merge");
  const FaceProjection proj = dim == 3 ? face_projection(q) : FaceProjection{};
  // node section layouts, bottom-up (node_section_layout, merge.cpp:751-762)
  g.sections.assign(n, {});
  for (int d = t.max_depth(); d >= 0; --d)
    for (int id : t.levels[d]) {
      auto& sec = g.sections[id];
      if (t.nch[id] == 0) {
        sec.assign(nf, Layout::panel(q, dim - 1));
        continue;
      }
      for (int f = 0; f < nf; ++f) {
        std::vector<Layout> quads(nquad);
        for (int c = 0; c < nc; ++c) {
          const int qp = ext_qpos(dim, c, f);
          if (qp >= 0) quads[qp] = g.sections[t.child[id][c]][f];
        }
        sec.push_back(Layout::split_of(std::move(quads)));
      }
    }
  auto nb_of = [&](int id) {
    int s = 0;
    for (const auto& l : g.sections[id]) s += l.npts();
    return s;
  };
  g.home.assign(n, {-1, -1, -1});
  // leaf groups by depth
  std::map<int, int> leaf_group_of_depth;
  for (int id : t.leaves) {
    auto it = leaf_group_of_depth.find(t.depth[id]);
    if (it == leaf_group_of_depth.end()) {
      it = leaf_group_of_depth.emplace(t.depth[id], int(g.leaf_groups.size())).first;
      LeafGroup lg;
      lg.depth = t.depth[id];
      lg.side = t.hi[3 * id] - t.lo[3 * id];
      g.leaf_groups.push_back(lg);
    }
    LeafGroup& lg = g.leaf_groups[it->second];
    g.home[id] = {0, it->second, int(lg.leaves.size())};
    lg.leaves.push_back(id);
  }
  const double pp = t.dim == 2 ? double(t.p) * t.p : double(t.p) * t.p * t.p;
  const double ni = t.dim == 2 ? double(q) * q : double(q) * q * q, nbl = 2.0 * dim * (dim == 2 ? q : q * q);
  const double ne = pp - ni;
  g.build_flops = t.leaves.size() *
                  (2.0 / 3.0 * ni * ni * ni + 2 * ni * ni * ne + 2 * ni * ne * nbl + 2 * nbl * pp * nbl + 2 * ni * ni +
                   2 * nbl * pp);
  // merge groups, deepest first
  g.merge_groups.assign(t.max_depth() + 1, {});
  for (int d = t.max_depth() - 1; d >= 0; --d) {
    std::map<std::string, int> by_key;
    for (int id : t.levels[d]) {
      if (t.nch[id] == 0) continue;
      std::string key;
      for (int c = 0; c < nc; ++c)
        for (int f = 0; f < nf; ++f) key += g.sections[t.child[id][c]][f].key() + ",";
      auto it = by_key.find(key);
      if (it != by_key.end()) {
        MergeGroup& mg = g.merge_groups[d][it->second];
        g.home[id] = {1, it->second, int(mg.nodes.size())};
        mg.nodes.push_back(id);
        continue;
      }
      by_key.emplace(key, int(g.merge_groups[d].size()));
      g.home[id] = {1, int(g.merge_groups[d].size()), 0};
      // ---- geometry of this signature (MergeGeom, merge.cpp:90-152)
      MergeGroup mg;
      mg.depth = d;
      mg.root = id == 0;
      mg.nodes.push_back(id);
      mg.nchild = nc;
      std::vector<std::array<int, 7>> coff(nc);
      for (int c = 0; c < nc; ++c) {
        const auto& sec = g.sections[t.child[id][c]];
        coff[c][0] = 0;
        for (int f = 0; f < nf; ++f) coff[c][f + 1] = coff[c][f] + sec[f].npts();
        mg.child_nb[c] = coff[c][nf];
      }
      std::vector<Layout> meets(ifs.size());
      std::vector<int> int_off(ifs.size());
      for (size_t k = 0; k < ifs.size(); ++k) {
        const Layout& la = g.sections[t.child[id][ifs[k].clo]][ifs[k].flo];
        const Layout& lb = g.sections[t.child[id][ifs[k].chi]][ifs[k].fhi];
        if (dim == 2 && la != lb)
          throw std::runtime_error(fmt("merge: interface layout mismatch at section %d (node %d)", int(k), id));
        if (dim == 3) {  // check_restriction (merge.cpp:74-87)
          std::function<void(const Layout&, const Layout&)> chk = [&](const Layout& a, const Layout& b) {
            if (!a.split && !b.split) return;
            if (!a.split || !b.split) {
              if ((a.split ? a : b).max_level() > 1)
                throw std::runtime_error(
                    "merge: level restriction violated at an interface; run enforce_level_restriction");
              return;
            }
            for (size_t i = 0; i < a.sub.size(); ++i) chk(a.sub[i], b.sub[i]);
          };
          chk(la, lb);
        }
        meets[k] = layout_meet(la, lb);
        int_off[k] = mg.n_int;
        mg.n_int += meets[k].npts();
      }
      // per (child, face): interface id or exterior offset (canonical parent order)
      std::vector<std::array<int, 6>> ext_off(nc), itf(nc);
      for (int c = 0; c < nc; ++c)
        for (int f = 0; f < nf; ++f) {
          ext_off[c][f] = -1;
          itf[c][f] = -1;
          for (size_t k = 0; k < ifs.size(); ++k)
            if ((ifs[k].clo == c && ifs[k].flo == f) || (ifs[k].chi == c && ifs[k].fhi == f)) itf[c][f] = int(k);
        }
      int pos = 0;
      for (int f = 0; f < nf; ++f) {
        std::vector<Layout> quads(nquad);
        std::vector<int> owner(nquad, -1);
        for (int c = 0; c < nc; ++c) {
          const int qp = ext_qpos(dim, c, f);
          if (qp < 0) continue;
          quads[qp] = g.sections[t.child[id][c]][f];
          owner[qp] = c;
        }
        for (int qv = 0; qv < nquad; ++qv) {
          ext_off[owner[qv]][f] = pos;
          pos += quads[qv].npts();
        }
        mg.sections.push_back(Layout::split_of(std::move(quads)));
      }
      mg.n_ext = pos;
      // transfers (row_tr / col_tr, merge.cpp:201-211) and the projected child layouts
      std::vector<std::array<HostMat, 6>> Rf(nc), Ef(nc);
      std::vector<std::array<int, 7>> coffp(nc);
      for (int c = 0; c < nc; ++c) {
        coffp[c][0] = 0;
        for (int f = 0; f < nf; ++f) {
          const Layout& lay = g.sections[t.child[id][c]][f];
          int len = lay.npts();
          if (itf[c][f] >= 0 && lay != meets[itf[c][f]]) {
            Rf[c][f] = layout_transfer(lay, meets[itf[c][f]], proj);
            Ef[c][f] = layout_transfer(meets[itf[c][f]], lay, proj);
            len = meets[itf[c][f]].npts();
            mg.proj[c] = true;
          }
          coffp[c][f + 1] = coffp[c][f] + len;
        }
        mg.child_nbp[c] = coffp[c][nf];
        if (mg.proj[c]) {  // full-size R (nbp x nb) and diag(1, E) ((1 + nb) x (1 + nbp))
          const int nb = mg.child_nb[c], nbp = mg.child_nbp[c];
          mg.R[c] = HostMat(nbp, nb);
          mg.Ehat[c] = HostMat(1 + nb, 1 + nbp);
          mg.Ehat[c](0, 0) = 1.0;
          for (int f = 0; f < nf; ++f) {
            const int r0 = coffp[c][f], c0 = coff[c][f], len0 = coff[c][f + 1] - c0, lenp = coffp[c][f + 1] - r0;
            if (Rf[c][f].r) {
              for (int j = 0; j < len0; ++j)
                for (int i = 0; i < lenp; ++i) {
                  mg.R[c](r0 + i, c0 + j) = Rf[c][f](i, j);
                  mg.Ehat[c](1 + c0 + j, 1 + r0 + i) = Ef[c][f](j, i);
                }
            } else {
              for (int i = 0; i < len0; ++i) {
                mg.R[c](r0 + i, c0 + i) = 1.0;
                mg.Ehat[c](1 + c0 + i, 1 + r0 + i) = 1.0;
              }
            }
          }
        }
      }
      // gather blocks on the projected children (merge.cpp:226-278)
      const bool need_ab = !mg.root;
      std::vector<BlockCopyG> first, second;
      for (int c = 0; c < nc; ++c)
        for (int rf = 0; rf < nf; ++rf) {
          const bool rext = ext_off[c][rf] >= 0;
          const int roff = rext ? ext_off[c][rf] : int_off[itf[c][rf]];
          const int rn = coffp[c][rf + 1] - coffp[c][rf];
          auto& pass = (!rext && ifs[itf[c][rf]].chi == c) ? second : first;
          // outgoing data: h_ext (AH column 0) or h_int (MD column n_int)
          if (rext) {
            if (need_ab) first.push_back({2, roff, 0, c, coffp[c][rf], 0, rn, 1});
          } else {
            pass.push_back({0, roff, mg.n_int, c, coffp[c][rf], 0, rn, 1});
          }
          for (int cf = 0; cf < nf; ++cf) {
            const bool cext = ext_off[c][cf] >= 0;
            const int coffs = cext ? ext_off[c][cf] : int_off[itf[c][cf]];
            const int cn = coffp[c][cf + 1] - coffp[c][cf];
            const int sr = coffp[c][rf], sc = 1 + coffp[c][cf];
            if (rext && cext) {
              if (need_ab) first.push_back({2, roff, 1 + coffs, c, sr, sc, rn, cn});
            } else if (rext) {
              if (need_ab) first.push_back({1, roff, coffs, c, sr, sc, rn, cn});
            } else if (cext) {
              pass.push_back({0, roff, mg.n_int + 1 + coffs, c, sr, sc, rn, cn});  // C (kept at an implicit root for the solve)
            } else {
              pass.push_back({0, roff, coffs, c, sr, sc, rn, cn});
            }
          }
        }
      mg.blocks = first;
      mg.pass_split = int(first.size());
      mg.blocks.insert(mg.blocks.end(), second.begin(), second.end());
      // downward maps (child_maps, merge.cpp:302-320)
      for (int c = 0; c < nc; ++c)
        for (int f = 0; f < nf; ++f) {
          DownCopy dc{};
          dc.child = c;
          dc.dst_off = coff[c][f];
          dc.dst_len = coff[c][f + 1] - coff[c][f];
          if (ext_off[c][f] >= 0) {
            dc.src_int = 0;
            dc.src_off = ext_off[c][f];
            dc.src_len = dc.dst_len;
            dc.E_off = -1;
          } else {
            const int k = itf[c][f];
            dc.src_int = 1;
            dc.src_off = int_off[k];
            dc.src_len = meets[k].npts();
            dc.E_off = -1;
            if (Ef[c][f].r) {
              dc.E_off = int(mg.Edata.size());
              mg.Edata.insert(mg.Edata.end(), Ef[c][f].a.begin(), Ef[c][f].a.end());
            }
          }
          mg.down.push_back(dc);
        }
      g.merge_groups[d].push_back(std::move(mg));
    }
    for (const MergeGroup& mg : g.merge_groups[d]) {
      const double a = mg.n_int, e = mg.n_ext;
      const double per = mg.root ? (implicit_root ? 2.0 / 3.0 * a * a * a : 2.0 / 3.0 * a * a * a + 2 * a * a * e)
                                 : 2.0 / 3.0 * a * a * a + 2 * a * a * e + 2 * e * a * e;
      g.build_flops += per * double(mg.nodes.size());
    }
  }
  g.root_nb = nb_of(0);
  g.top_D = g.merge_groups[0][0].n_int;
  return g;
}

// ---------------------------------------------------------------- adaptive refinement
namespace {
struct MutTree {  // DiscretizationTree while it grows (split / finalize / find_node, mesh.cpp:27-88)
  GTree& t;
  std::vector<long long>& anchor;
  void split(int id) {
    const int nc = t.nchild;
    t.nch[id] = nc;
    for (int c = 0; c < nc; ++c) {
      const int k = int(t.depth.size());
      t.depth.push_back(t.depth[id] + 1);
      t.nch.push_back(0);
      t.child.push_back({-1, -1, -1, -1, -1, -1, -1, -1});
      t.child[id][c] = k;
      for (int a = 0; a < 3; ++a) {
        const double mid = 0.5 * (t.lo[3 * id + a] + t.hi[3 * id + a]);
        const bool hi_half = a < t.dim && kOff[c][a];
        t.lo.push_back(hi_half ? mid : t.lo[3 * id + a]);
        t.hi.push_back(a < t.dim && !kOff[c][a] ? mid : t.hi[3 * id + a]);
        anchor.push_back(a < t.dim ? 2 * anchor[3 * id + a] + kOff[c][a] : 0);
      }
    }
  }
  void finalize() {
    t.levels.clear();
    t.leaves.clear();
    std::vector<int> stack{0};
    while (!stack.empty()) {
      const int id = stack.back();
      stack.pop_back();
      if ((int)t.levels.size() <= t.depth[id]) t.levels.resize(t.depth[id] + 1);
      t.levels[t.depth[id]].push_back(id);
      if (t.nch[id] == 0)
        t.leaves.push_back(id);
      else
        for (int c = t.nchild - 1; c >= 0; --c) stack.push_back(t.child[id][c]);
    }
  }
  int find_node(int depth, const long long* a) const {
    const long long lim = 1LL << depth;
    for (int k = 0; k < t.dim; ++k)
      if (a[k] < 0 || a[k] >= lim) return -1;
    int id = 0;
    for (int level = 1; level <= depth; ++level) {
      if (t.nch[id] == 0) return id;
      const int shift = depth - level;
      const int o1 = int((a[0] >> shift) & 1), o2 = int((a[1] >> shift) & 1);
      const int o3 = t.dim == 3 ? int((a[2] >> shift) & 1) : 0;
      static const int slot2[2][2] = {{0, 3}, {1, 2}};
      id = t.child[id][slot2[o1][o2] + 4 * o3];
    }
    return id;
  }
  int max_leaf_depth_on_face(int id, int axis, int sign) const {
    if (t.nch[id] == 0) return t.depth[id];
    int best = 0;
    for (int c = 0; c < t.nchild; ++c)
      if (kOff[c][axis] == (sign > 0 ? 1 : 0)) best = std::max(best, max_leaf_depth_on_face(t.child[id][c], axis, sign));
    return best;
  }
};

void level_restrict(MutTree& m) {
  GTree& t = m.t;
  bool changed = true;
  while (changed) {
    changed = false;
    m.finalize();
    const std::vector<int> snapshot = t.leaves;
    for (int id : snapshot) {
      if (t.nch[id] != 0) continue;
      const int depth = t.depth[id];
      long long an[3] = {m.anchor[3 * id], m.anchor[3 * id + 1], m.anchor[3 * id + 2]};
      for (int axis = 0; axis < t.dim && t.nch[id] == 0; ++axis)
        for (int sign = -1; sign <= 1; sign += 2) {
          long long na[3] = {an[0], an[1], an[2]};
          na[axis] += sign;
          const int nb = m.find_node(depth, na);
          if (nb < 0 || t.depth[nb] < depth) continue;
          if (m.max_leaf_depth_on_face(nb, axis, -sign) > depth + 1) {
            m.split(id);
            changed = true;
            break;
          }
        }
    }
  }
  m.finalize();
}

HostMat refinement_interpolant(int p) {  // spectral.cpp:438-452, octants (a..h), tensor (i1 p + i2) p + i3
  const std::vector<double> cn = cheb_nodes(p);
  std::vector<double> lo(p), hi(p);
  for (int i = 0; i < p; ++i) lo[i] = (cn[i] - 1.0) / 2.0, hi[i] = (cn[i] + 1.0) / 2.0;
  const HostMat e[2] = {bary_interp(cn, lo), bary_interp(cn, hi)};
  const int pc = p * p * p;
  HostMat out(8 * pc, pc);
  for (int c = 0; c < 8; ++c)
    for (int i1 = 0; i1 < p; ++i1)
      for (int i2 = 0; i2 < p; ++i2)
        for (int i3 = 0; i3 < p; ++i3)
          for (int j1 = 0; j1 < p; ++j1)
            for (int j2 = 0; j2 < p; ++j2)
              for (int j3 = 0; j3 < p; ++j3)
                out(c * pc + (i1 * p + i2) * p + i3, (j1 * p + j2) * p + j3) =
                    e[kOff[c][0]](i1, j1) * (e[kOff[c][1]](i2, j2) * e[kOff[c][2]](i3, j3));
  return out;
}

struct FieldRefiner {  // mesh.cpp:171-229
  PointField f;
  const void* ctx;
  const HostMat* l8f1;
  int p;
  double tol, sup;
  int max_depth;
  std::set<std::pair<int, std::array<long long, 3>>> accepted, want_split;

  std::vector<double> sample(const double* lo, const double* hi) const {
    const std::vector<double> cn = cheb_nodes(p);
    std::vector<double> v;
    v.reserve(size_t(p) * p * p);
    auto map1 = [&](double s, int k) { return 0.5 * (lo[k] + hi[k]) + 0.5 * (hi[k] - lo[k]) * s; };
    for (int i1 = 0; i1 < p; ++i1)
      for (int i2 = 0; i2 < p; ++i2)
        for (int i3 = 0; i3 < p; ++i3) {
          const double x[3] = {map1(cn[i1], 0), map1(cn[i2], 1), map1(cn[i3], 2)};
          const double y = f(ctx, x);
          if (!std::isfinite(y)) throw std::runtime_error("refine_adaptive: non-finite field sample");
          v.push_back(y);
        }
    return v;
  }
  static void child_box(const double* lo, const double* hi, int c, double* clo, double* chi) {
    for (int k = 0; k < 3; ++k) {
      const double mid = 0.5 * (lo[k] + hi[k]);
      clo[k] = kOff[c][k] ? mid : lo[k];
      chi[k] = kOff[c][k] ? hi[k] : mid;
    }
  }
  double check(const double* lo, const double* hi, const std::vector<double>& x0, std::vector<double>& x1) {
    const int pc = p * p * p;
    x1.assign(size_t(8) * pc, 0.0);
    for (int c = 0; c < 8; ++c) {
      double clo[3], chi[3];
      child_box(lo, hi, c, clo, chi);
      const std::vector<double> s = sample(clo, chi);
      std::copy(s.begin(), s.end(), x1.begin() + size_t(c) * pc);
    }
    for (double v : x0) sup = std::max(sup, std::abs(v));
    for (double v : x1) sup = std::max(sup, std::abs(v));
    std::vector<double> y(size_t(8) * pc, 0.0);  // L8f1 x0, column sweep (column-major)
    for (int j = 0; j < pc; ++j) {
      const double xj = x0[j];
      const double* col = &l8f1->a[size_t(j) * 8 * pc];
      for (int i = 0; i < 8 * pc; ++i) y[i] += col[i] * xj;
    }
    double err = 0.0;
    for (int i = 0; i < 8 * pc; ++i) err = std::max(err, std::abs(x1[i] - y[i]));
    return err;
  }
  void refine(const double* lo, const double* hi, int depth, const std::array<long long, 3>& an,
              const std::vector<double>& x0) {
    std::vector<double> x1;
    const double err = check(lo, hi, x0, x1);
    if (err / sup < tol) {
      accepted.insert({depth, an});
      return;
    }
    if (depth >= max_depth) return;
    want_split.insert({depth, an});
    const int pc = p * p * p;
    for (int c = 0; c < 8; ++c) {
      std::array<long long, 3> ca;
      for (int k = 0; k < 3; ++k) ca[k] = 2 * an[k] + kOff[c][k];
      double clo[3], chi[3];
      child_box(lo, hi, c, clo, chi);
      refine(clo, chi, depth + 1, ca, std::vector<double>(x1.begin() + size_t(c) * pc, x1.begin() + size_t(c + 1) * pc));
    }
  }
};
}  // namespace

void enforce_level_restriction(GTree& t, std::vector<long long>& anchor) {
  MutTree m{t, anchor};
  level_restrict(m);
  finalize_gtree(t);
}

RefineResult refine_adaptive(const double* lo, const double* hi, int p, double tol, int max_depth,
                             const std::vector<std::pair<PointField, const void*>>& fields) {
  if (fields.empty()) throw std::runtime_error("refine_adaptive: no test fields");
  if (!(tol > 0)) throw std::runtime_error("refine_adaptive: tol must be positive");
  const HostMat l8f1 = refinement_interpolant(p);
  RefineResult res;
  GTree& t = res.tree;
  t.dim = 3;
  t.p = p;
  t.nchild = 8;
  t.nface = 6;
  t.depth = {0};
  t.nch = {0};
  t.child = {{-1, -1, -1, -1, -1, -1, -1, -1}};
  t.lo.assign(lo, lo + 3);
  t.hi.assign(hi, hi + 3);
  res.anchor = {0, 0, 0};
  MutTree m{t, res.anchor};
  // phase 1: independent per-field refinement
  // (decisions for one field never depend on another field's samples, mesh.cpp:250-252: one host thread
  // per field; the union below is order-independent)
  std::vector<FieldRefiner> refiners(fields.size());
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(fields.size());
  for (size_t f = 0; f < fields.size(); ++f) {
    FieldRefiner& r = refiners[f];
    r.f = fields[f].first;
    r.ctx = fields[f].second;
    r.l8f1 = &l8f1;
    r.p = p;
    r.tol = tol;
    r.sup = 0.0;
    r.max_depth = max_depth;
    pool.emplace_back([&r, &errs, f, lo, hi] {
      try {
        r.refine(lo, hi, 0, {0, 0, 0}, r.sample(lo, hi));
      } catch (...) {
        errs[f] = std::current_exception();
      }
    });
  }
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
  // union of the per-field trees
  std::set<std::pair<int, std::array<long long, 3>>> splits;
  for (const auto& r : refiners) splits.insert(r.want_split.begin(), r.want_split.end());
  bool grew = true;
  while (grew) {
    grew = false;
    m.finalize();
    const std::vector<int> lv = t.leaves;
    for (int id : lv)
      if (splits.count({t.depth[id], {res.anchor[3 * id], res.anchor[3 * id + 1], res.anchor[3 * id + 2]}})) {
        m.split(id);
        grew = true;
      }
  }
  // phase 2: level restriction + verification of every leaf against every field
  bool changed = true;
  while (changed) {
    changed = false;
    level_restrict(m);
    const std::vector<int> lv = t.leaves;
    for (int id : lv) {
      if (t.nch[id] != 0) continue;
      if (t.depth[id] >= max_depth) continue;
      const std::array<long long, 3> an{res.anchor[3 * id], res.anchor[3 * id + 1], res.anchor[3 * id + 2]};
      for (auto& r : refiners) {
        if (r.accepted.count({t.depth[id], an})) continue;
        std::vector<double> x1;
        const std::vector<double> x0 = r.sample(&t.lo[3 * id], &t.hi[3 * id]);
        if (r.check(&t.lo[3 * id], &t.hi[3 * id], x0, x1) / r.sup < tol) {
          r.accepted.insert({t.depth[id], an});
          continue;
        }
        m.split(id);
        changed = true;
        break;
      }
    }
    if (changed) m.finalize();
  }
  for (int id : t.leaves) {
    if (t.depth[id] < max_depth) continue;
    for (auto& r : refiners) {
      std::vector<double> x1;
      const std::vector<double> x0 = r.sample(&t.lo[3 * id], &t.hi[3 * id]);
      if (r.check(&t.lo[3 * id], &t.hi[3 * id], x0, x1) / r.sup >= tol) {
        res.unresolved.push_back(id);
        break;
      }
    }
  }
  for (const auto& r : refiners) res.global_sup.push_back(r.sup);
  finalize_gtree(t);
  return res;
}

// ---------------------------------------------------------------- points
namespace {
void collect(const double* lo0, const double* hi0, int dim, int face, const Layout& lay, const std::vector<double>& gx,
             std::vector<double>& out) {
  double lo[3] = {lo0[0], lo0[1], lo0[2]}, hi[3] = {hi0[0], hi0[1], hi0[2]};
  const int q = lay.q;
  auto map1 = [&](double t, int k) { return 0.5 * (lo[k] + hi[k]) + 0.5 * (hi[k] - lo[k]) * t; };
  if (!lay.split) {  // proj/src/mesh.cpp:342-380 restricted to this face
    if (dim == 2) {
      for (int i = 0; i < q; ++i) {
        double x[3] = {0, 0, 0};
        switch (face) {
          case 0: x[0] = map1(gx[i], 0); x[1] = lo[1]; break;
          case 1: x[0] = hi[0]; x[1] = map1(gx[i], 1); break;
          case 2: x[0] = map1(gx[i], 0); x[1] = hi[1]; break;
          default: x[0] = lo[0]; x[1] = map1(gx[i], 1); break;
        }
        out.insert(out.end(), x, x + 3);
      }
    } else {
      const int axis = face / 2, ua = axis == 0 ? 1 : 0, va = axis == 2 ? 1 : 2;
      const double fixed = face % 2 == 0 ? lo[axis] : hi[axis];
      for (int iu = 0; iu < q; ++iu)
        for (int iv = 0; iv < q; ++iv) {
          double x[3];
          x[axis] = fixed;
          x[ua] = map1(gx[iu], ua);
          x[va] = map1(gx[iv], va);
          out.insert(out.end(), x, x + 3);
        }
    }
    return;
  }
  double mid[3];
  for (int k = 0; k < 3; ++k) mid[k] = 0.5 * (lo[k] + hi[k]);
  if (dim == 2) {  // proj/src/layout.cpp:100-107
    const int axis = (face == 0 || face == 2) ? 0 : 1;
    for (int h = 0; h < 2; ++h) {
      double sl[3] = {lo[0], lo[1], lo[2]}, sh[3] = {hi[0], hi[1], hi[2]};
      (h ? sl : sh)[axis] = mid[axis];
      collect(sl, sh, dim, face, lay.sub[h], gx, out);
    }
  } else {  // :108-118
    const int fa = face / 2, ua = fa == 0 ? 1 : 0, va = fa == 2 ? 1 : 2;
    for (int hu = 0; hu < 2; ++hu)
      for (int hv = 0; hv < 2; ++hv) {
        double sl[3] = {lo[0], lo[1], lo[2]}, sh[3] = {hi[0], hi[1], hi[2]};
        (hu ? sl : sh)[ua] = mid[ua];
        (hv ? sl : sh)[va] = mid[va];
        collect(sl, sh, dim, face, lay.sub[hu * 2 + hv], gx, out);
      }
  }
}
}  // namespace

std::vector<double> general_root_points(const GeneralPlan& g) {
  std::vector<double> gx, gw;
  gauss_rule(g.tree.q, gx, gw);
  std::vector<double> out;
  for (int f = 0; f < g.tree.nface; ++f) collect(&g.tree.lo[0], &g.tree.hi[0], g.tree.dim, f, g.sections[0][f], gx, out);
  return out;
}

void general_leaf_points_into(const GeneralPlan& g, double* out) {
  const GTree& t = g.tree;
  const std::vector<double> cn = cheb_nodes(t.p);
  const int np = t.dim == 2 ? t.p * t.p : t.p * t.p * t.p;
  std::vector<double> m(size_t(3 * t.p));
  for (size_t l = 0; l < t.leaves.size(); ++l) {
    const int id = t.leaves[l];
    const double* lo = &t.lo[3 * id];
    const double* hi = &t.hi[3 * id];
    for (int k = 0; k < 3; ++k)  // per-axis mapped nodes, same expression as leaf_cheb_points
      for (int i = 0; i < t.p; ++i) m[size_t(k * t.p + i)] = 0.5 * (lo[k] + hi[k]) + 0.5 * (hi[k] - lo[k]) * cn[size_t(i)];
    double* o = out + l * size_t(np) * 3;
    if (t.dim == 2) {
      for (int i1 = 0; i1 < t.p; ++i1)
        for (int i2 = 0; i2 < t.p; ++i2, o += 3) o[0] = m[size_t(i1)], o[1] = m[size_t(t.p + i2)], o[2] = 0.0;
    } else {
      for (int i1 = 0; i1 < t.p; ++i1)
        for (int i2 = 0; i2 < t.p; ++i2)
          for (int i3 = 0; i3 < t.p; ++i3, o += 3)
            o[0] = m[size_t(i1)], o[1] = m[size_t(t.p + i2)], o[2] = m[size_t(2 * t.p + i3)];
    }
  }
}

std::vector<double> general_leaf_points(const GeneralPlan& g) {
  const GTree& t = g.tree;
  const size_t np = t.dim == 2 ? size_t(t.p) * t.p : size_t(t.p) * t.p * t.p;
  std::vector<double> out(t.leaves.size() * np * 3);
  general_leaf_points_into(g, out.data());
  return out;
}

}  // namespace hpsg
