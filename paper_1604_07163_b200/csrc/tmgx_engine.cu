// Host orchestration of the MG-CG path; see tmgx_engine.hpp for the reference map.
#include "tmgx_engine.hpp"

#include <chrono>

#include <algorithm>
#include <cmath>
#include <cstring>

namespace tmgx {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw tmg::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

// ------------------------------------------------------------------------------------------
// World
// ------------------------------------------------------------------------------------------

Owners::Owners(int R_, int P_, int me_) : R(R_), P(P_), me(me_) {
  if (R < 1 || P < 1 || me < 0 || me >= P || R < P)
    throw tmg::ConfigError("world: need n_ranks >= nproc >= 1 and 0 <= proc < nproc");
  first = (int)((long long)me * R / P);
  end = (int)((long long)(me + 1) * R / P);
}

World::World(int R_, int P_, int me_, int device_, const char* job) : Owners(R_, P_, me_), device(device_) {
  CK(cudaSetDevice(device));
  CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  if (P > 1) {
    if (!job || !*job) throw tmg::ConfigError("world: nproc > 1 needs a job token (the node-local rendezvous name)");
    grp = std::make_unique<NodeGroup>(job, P, me);
  }
}

World::~World() {
  grp.reset();
  if (stream) cudaStreamDestroy(stream);
}

void World::stream_barrier() {
  grp->enqueue_barrier(stream);
  ++nbar;
}

void World::check() const {
  if (grp && grp->failed()) throw tmg::CudaError("world: a stream barrier timed out or a peer process aborted");
}

int Owners::owner(int wr) const {
  for (int p = 0; p < P; ++p)
    if (wr < (int)((long long)(p + 1) * R / P)) return p;
  return P - 1;
}

// ------------------------------------------------------------------------------------------
// Dist / Field / arena
// ------------------------------------------------------------------------------------------

int Dist::slot_of(int m) const {
  for (size_t q = 0; q < local.size(); ++q)
    if (local[q] == m) return (int)q;
  return -1;
}

long long Dist::local_unknowns() const {
  long long n = 0;
  for (const auto& g : geo) n += (long long)g.ex * g.ey * g.ez;
  return n;
}

static BoxGeo make_geo(const tmg::GridHeader& h, int m) {
  const tmg::GridBox b = h.box(m);
  BoxGeo g;
  g.ex = (int)b.extent(0);
  g.ey = (int)b.extent(1);
  g.ez = (int)b.extent(2);
  g.gx = (int)b.lo[0];
  g.gy = (int)b.lo[1];
  g.gz = (int)b.lo[2];
  g.Nx = (int)h.npoints[0];
  g.Ny = (int)h.npoints[1];
  g.Nz = (int)h.npoints[2];
  static const long long min_blocks = [] {  // TMGX_MIN_BLOCKS: tuning experiments
    const char* e = std::getenv("TMGX_MIN_BLOCKS");
    return e ? std::atoll(e) : (long long)kMinBlocks;
  }();
  g.zc = choose_zc(g.ex, g.ey, g.ez, min_blocks);
  g.px =((kXO + g.ex + 1) + 3) / 4 * 4;
  g.pxy = g.px * (g.ey + 2);
  g.base = kXO + g.px + g.pxy;
  g.total = g.pxy * (g.ez + 2) + 8;
  return g;
}

static long long geo_off(const BoxGeo& g, long long i, long long j, long long k) {
  return g.base + (i - g.gx) + g.px * (j - g.gy) + g.pxy * (k - g.gz);
}

std::shared_ptr<Dist> make_dist(const Owners& W, const tmg::GridHeader& h, const std::vector<int>& wr) {
  auto D = std::make_shared<Dist>();
  D->h = h;
  D->wr = wr;
  if ((int)wr.size() != h.n_ranks()) throw tmg::Error("dist: rank map does not match the header");
  for (int m = 0; m < h.n_ranks(); ++m)
    if (W.local(wr[m])) {
      D->local.push_back(m);
      D->geo.push_back(make_geo(h, m));
    }
  if ((int)D->local.size() > kMaxLocal) throw tmg::ConfigError("too many boxes per process");
  return D;
}

PtrTable Field::table() const {
  PtrTable t{};
  for (size_t q = 0; q < p.size() && q < (size_t)kMaxLocal; ++q) t.p[q] = p[q];
  return t;
}

DeviceArena::~DeviceArena() {
  for (void* p : ptrs_) cudaFree(p);
}

double* DeviceArena::alloc(long long n) {
  void* p = nullptr;
  if (n < 1) n = 1;
  if (!stream_) throw tmg::Error("device arena: no stream bound");
  CK(cudaMalloc(&p, (size_t)n * sizeof(double)));
  ptrs_.push_back(p);
  CK(cudaMemsetAsync(p, 0, (size_t)n * sizeof(double), stream_));
  return static_cast<double*>(p);
}

void DeviceArena::upload(void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream_));
  CK(cudaStreamSynchronize(stream_));
}

Field make_field(DeviceArena& A, const Dist& D) {
  Field f;
  for (const auto& g : D.geo) f.p.push_back(A.alloc(g.total));
  return f;
}

// ------------------------------------------------------------------------------------------
// Region plans
// ------------------------------------------------------------------------------------------

namespace {

// checksum of the global vertex indices of a region (both ends compute it from the headers)
unsigned long long region_sum(const tmg::GridBox& reg, const tmg::GridHeader& h) {
  unsigned long long s = 0;
  for (long long k = reg.lo[2]; k < reg.hi[2]; ++k)
    for (long long j = reg.lo[1]; j < reg.hi[1]; ++j)
      for (long long i = reg.lo[0]; i < reg.hi[0]; ++i) {
        const unsigned long long nat = (unsigned long long)(i + h.npoints[0] * (j + h.npoints[1] * k));
        s = s * 1099511628211ULL + (nat ^ 0x9e3779b97f4a7c15ULL);
      }
  return s;
}

template <class RegionFn>
PlanHost plan_host(const Owners& W, const Dist& S, const Dist& T, RegionFn region) {
  PlanHost plan;
  std::vector<long long> scount(W.P, 0), rcount(W.P, 0);
  // pass 1: count per peer
  for (int m = 0; m < T.h.n_ranks(); ++m)
    for (int s = 0; s < S.h.n_ranks(); ++s) {
      tmg::GridBox reg;
      if (!region(s, m, reg)) continue;
      const int os = W.owner(S.wr[s]), ot = W.owner(T.wr[m]);
      if (os == ot) continue;
      if (os == W.me) scount[ot] += reg.n_vertices();
      if (ot == W.me) rcount[os] += reg.n_vertices();
    }
  std::vector<long long> soff(W.P, 0), roff(W.P, 0);
  std::vector<int> sidx(W.P, -1), ridx(W.P, -1);
  for (int p = 0; p < W.P; ++p) {
    soff[p] = plan.send_total;
    roff[p] = plan.recv_total;
    if (scount[p]) {
      sidx[p] = (int)plan.sends.size();
      plan.sends.push_back({p, plan.send_total, scount[p]});
      plan.send_sum.push_back(0);
    }
    if (rcount[p]) {
      ridx[p] = (int)plan.recvs.size();
      plan.recvs.push_back({p, plan.recv_total, rcount[p]});
      plan.recv_sum.push_back(0);
    }
    plan.send_total += scount[p];
    plan.recv_total += rcount[p];
  }
  // pass 2: descriptors in (m asc, s asc) order, identical on both sides of every pair
  for (int m = 0; m < T.h.n_ranks(); ++m)
    for (int s = 0; s < S.h.n_ranks(); ++s) {
      tmg::GridBox reg;
      if (!region(s, m, reg)) continue;
      const int os = W.owner(S.wr[s]), ot = W.owner(T.wr[m]);
      if (os != W.me && ot != W.me) continue;
      CopyDesc d{};
      d.nx = (int)reg.extent(0);
      d.ny = (int)reg.extent(1);
      d.nz = (int)reg.extent(2);
      const long long n = reg.n_vertices();
      if (os == W.me) {
        const int ss = S.slot_of(s);
        const BoxGeo& gs = S.geo[ss];
        d.src_slot = ss;
        d.src_off = geo_off(gs, reg.lo[0], reg.lo[1], reg.lo[2]);
        d.src_px = gs.px;
        d.src_pxy = gs.pxy;
      }
      if (ot == W.me) {
        const int ts = T.slot_of(m);
        const BoxGeo& gt = T.geo[ts];
        d.dst_slot = ts;
        d.dst_off = geo_off(gt, reg.lo[0], reg.lo[1], reg.lo[2]);
        d.dst_px = gt.px;
        d.dst_pxy = gt.pxy;
      }
      if (os == W.me && ot == W.me) {
        plan.loc.push_back(d);
        plan.local_count += n;
        plan.max_local = std::max<long long>(plan.max_local, n);
      } else if (os == W.me) {
        d.dst_slot = -1;
        d.dst_off = soff[ot];
        d.dst_px = d.nx;
        d.dst_pxy = (long long)d.nx * d.ny;
        soff[ot] += n;
        plan.pack.push_back(d);
        plan.pack_peer.push_back(ot);
        plan.max_pack = std::max<long long>(plan.max_pack, n);
        auto& cs = plan.send_sum[sidx[ot]];
        cs = cs * 31 + region_sum(reg, T.h);
      } else {
        d.src_slot = -1;
        d.src_off = roff[os];
        d.src_px = d.nx;
        d.src_pxy = (long long)d.nx * d.ny;
        roff[os] += n;
        plan.unpack.push_back(d);
        plan.max_unpack = std::max<long long>(plan.max_unpack, n);
        auto& cs = plan.recv_sum[ridx[os]];
        cs = cs * 31 + region_sum(reg, T.h);
      }
    }
  return plan;
}

}  // namespace

RegionPlan upload_plan(DeviceArena& A, const PlanHost& h) {
  RegionPlan plan;
  auto up = [&](const std::vector<CopyDesc>& v, CopyDesc*& dst, int& n) {
    n = (int)v.size();
    if (!n) return;
    dst = A.alloc_t<CopyDesc>(n);
    A.upload(dst, v.data(), sizeof(CopyDesc) * v.size());
  };
  up(h.loc, plan.d_local, plan.n_local);
  up(h.pack, plan.d_pack, plan.n_pack);  // rewired to peer mailboxes by Solver::wire_transport
  up(h.unpack, plan.d_unpack, plan.n_unpack);
  plan.max_local = h.max_local;
  plan.max_pack = h.max_pack;
  plan.max_unpack = h.max_unpack;
  plan.sends = h.sends;
  plan.recvs = h.recvs;
  plan.send_total = h.send_total;
  plan.recv_total = h.recv_total;
  plan.pack_h = h.pack;
  plan.pack_peer = h.pack_peer;
  return plan;
}

// A plan moving `ncomp` consecutive component planes (component c of a box at p + c * total) in one
// use: every region descriptor repeated per component; each peer segment of the packed buffer
// holds its regions component-major (segment offset and size scaled by ncomp, identical on both
// ends), so a cross-process exchange of all components costs one publishing barrier.
PlanHost expand_components(const PlanHost& h, const Dist& S, const Dist& T, int ncomp) {
  if (ncomp == 1) return h;
  PlanHost o = h;
  o.loc.clear();
  o.pack.clear();
  o.unpack.clear();
  o.pack_peer.clear();
  for (auto& sd : o.sends) sd.off *= ncomp, sd.count *= ncomp;
  for (auto& rv : o.recvs) rv.off *= ncomp, rv.count *= ncomp;
  o.send_total *= ncomp;
  o.recv_total *= ncomp;
  o.local_count *= ncomp;
  auto seg_of = [](const std::vector<RegionPlan::Peer>& v, long long off) -> const RegionPlan::Peer& {
    for (const auto& e : v)
      if (off >= e.off && off < e.off + e.count) return e;
    throw tmg::Error("plan: packed offset outside every peer segment");
  };
  for (int c = 0; c < ncomp; ++c) {
    for (const CopyDesc& d : h.loc) {
      CopyDesc e = d;
      e.src_off += c * S.geo[(size_t)d.src_slot].total;
      e.dst_off += c * T.geo[(size_t)d.dst_slot].total;
      o.loc.push_back(e);
    }
    for (size_t k = 0; k < h.pack.size(); ++k) {
      const CopyDesc& d = h.pack[k];
      const RegionPlan::Peer& sg = seg_of(h.sends, d.dst_off);
      CopyDesc e = d;
      e.src_off += c * S.geo[(size_t)d.src_slot].total;
      e.dst_off = sg.off * ncomp + c * sg.count + (d.dst_off - sg.off);
      o.pack.push_back(e);
      o.pack_peer.push_back(h.pack_peer[k]);
    }
    for (const CopyDesc& d : h.unpack) {
      const RegionPlan::Peer& sg = seg_of(h.recvs, d.src_off);
      CopyDesc e = d;
      e.src_off = sg.off * ncomp + c * sg.count + (d.src_off - sg.off);
      e.dst_off += c * T.geo[(size_t)d.dst_slot].total;
      o.unpack.push_back(e);
    }
  }
  return o;
}

// ghost_exchange (grid.cpp:645-696): every rank's halo box (width 1, clipped to the grid,
// edges and corners included) is filled from the owning boxes.
PlanHost halo_plan_host(const Owners& W, const Dist& D) {
  return plan_host(W, D, D, [&](int s, int m, tmg::GridBox& reg) {
    if (s == m) return false;
    tmg::GridBox hb = D.h.box(m);
    for (int a = 0; a < 3; ++a) {
      hb.lo[a] = std::max<long long>(0, hb.lo[a] - 1);
      hb.hi[a] = std::min<long long>(D.h.npoints[a], hb.hi[a] + 1);
    }
    reg = tmg::intersect(hb, D.h.box(s));
    return !reg.empty();
  });
}

// P-hat^T composed with ScatterPlan::to_sub (grid.cpp:582-599, scatter_plan.cpp:40-77):
// every vertex moves from its parent owner box to the member box that owns it in the
// repartitioned header, i.e. box intersections of the two decompositions.
PlanHost transfer_plan_host(const Owners& W, const Dist& S, const Dist& T) {
  return plan_host(W, S, T, [&](int s, int m, tmg::GridBox& reg) {
    reg = tmg::intersect(S.h.box(s), T.h.box(m));
    return !reg.empty();
  });
}

// One use of a plan. Cross-process regions: pack straight into the peers' mailboxes, one stream
// barrier publishes them, unpack from this process's mailbox. A plan reused with no barrier since
// its previous use first waits for the peers to have unpacked that use (write-after-read).
void run_plan(World& W, RegionPlan& plan, const Field& src, const Field& dst, bool telescope) {
  const PtrTable ts = src.table(), td = dst.table();
  const bool xp = plan.xproc && W.P > 1;
  if (xp && plan.last_bar == W.nbar) W.stream_barrier();
  if (plan.n_pack) {
    W.cnt.launches += launch_region_copy(plan.d_pack, plan.n_pack, plan.max_pack, ts, td, nullptr, nullptr, W.stream);
    (telescope ? W.cnt.tele_bytes : W.cnt.halo_bytes) += plan.send_total * 8;
  }
  if (plan.n_local)
    W.cnt.launches += launch_region_copy(plan.d_local, plan.n_local, plan.max_local, ts, td, nullptr, nullptr, W.stream);
  if (xp) {
    W.stream_barrier();
    plan.last_bar = W.nbar;
  }
  if (plan.n_unpack)
    W.cnt.launches += launch_region_copy(plan.d_unpack, plan.n_unpack, plan.max_unpack, ts, td, plan.recvbuf, nullptr,
                                         W.stream);
}

// ------------------------------------------------------------------------------------------
// Solver setup
// ------------------------------------------------------------------------------------------

unsigned long long splitmix64_h(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
double hashed_uniform_h(unsigned long long seed, unsigned long long idx) {
  return (double)(splitmix64_h(seed ^ splitmix64_h(idx)) >> 11) * 0x1.0p-53;
}
static double harm_h(double a, double b) { return 2.0 * a * b / (a + b); }

double Solver::host_k(const Dist& D, long long gi, long long gj, long long gk) const {
  if (prob.kind != 1) return 1.0;
  volatile double x = (double)gi * (1.0 / (double)(D.h.npoints[0] - 1));
  volatile double y = (double)gj * (1.0 / (double)(D.h.npoints[1] - 1));
  volatile double z = (double)gk * (1.0 / (double)(D.h.npoints[2] - 1));
  for (const Sphere& s : spheres) {
    volatile double dx = x - s.cx, dy = y - s.cy, dz = z - s.cz;
    volatile double a = dx * dx, b = dy * dy, c = dz * dz;
    volatile double ab = a + b;
    volatile double d2 = ab + c;
    volatile double rr = s.r * s.r;
    if (d2 <= rr) return prob.k_in;
  }
  return 1.0;
}

static OpParams make_op(const tmg::GridHeader& h) {
  OpParams op{};
  double ih2[3];
  for (int a = 0; a < 3; ++a) {
    const double hh = 1.0 / (double)(h.npoints[a] - 1);
    ih2[a] = 1.0 / (hh * hh);
  }
  op.ih2x = ih2[0];
  op.ih2y = ih2[1];
  op.ih2z = ih2[2];
  volatile double d = 0.0;  // oracle order: -z,-y,-x,+x,+y,+z
  d = d + ih2[2];
  d = d + ih2[1];
  d = d + ih2[0];
  d = d + ih2[0];
  d = d + ih2[1];
  d = d + ih2[2];
  op.cdiag = d;
  op.cinvd = 1.0 / op.cdiag;
  op.k = nullptr;
  return op;
}

Solver::Solver(World& W_, const ProblemDesc& P, const MGDesc& M) : W(W_), prob(P), mgd(M) {
  CK(cudaSetDevice(W.device));
  arena.set_stream(W.stream);
  if (const char* e = std::getenv("TMGX_GRAPHS")) use_graphs = std::string(e) != "0";
  if (const char* e = std::getenv("TMGX_TB")) tb_enabled = std::string(e) != "0";
  if (const char* e = std::getenv("TMGX_FUSE_CG")) fuse_cg = std::string(e) != "0";
  if (const char* e = std::getenv("TMGX_TB_MIN")) tb_min_extent = std::atoi(e);
  if (const char* e = std::getenv("TMGX_TB3")) tb3_enabled = std::string(e) != "0";
  if (const char* e = std::getenv("TMGX_FUSE_DOTS")) fuse_dots = std::string(e) != "0";
  if (const char* e = std::getenv("TMGX_FUSE_RR")) fuse_rr = std::string(e) != "0";
  if (const char* e = std::getenv("TMGX_FUSE_RR2")) fuse_rr2 = std::atoi(e);
  if (const char* e = std::getenv("TMGX_CC_MAX")) cc_max_extent = std::atoi(e);
  if (mgd.nlevels < 1) throw tmg::ConfigError("mg: number of levels must be >= 1");
  if (mgd.m < 1) throw tmg::ConfigError("mg: smoother iterations must be >= 1");
  if (prob.kind == 1) {
    // sphere s: centre u(seed,4s+0..2), radius 0.05 + 0.10 u(seed,4s+3)
    for (int s = 0; s < prob.n_spheres; ++s) {
      Sphere sp;
      sp.cx = hashed_uniform_h(prob.seed_k, 4ull * s + 0);
      sp.cy = hashed_uniform_h(prob.seed_k, 4ull * s + 1);
      sp.cz = hashed_uniform_h(prob.seed_k, 4ull * s + 2);
      sp.r = 0.05 + 0.10 * hashed_uniform_h(prob.seed_k, 4ull * s + 3);
      spheres.push_back(sp);
    }
    spheres_dev = arena.alloc_t<Sphere>((long long)spheres.size());
    arena.upload(spheres_dev, spheres.data(), sizeof(Sphere) * spheres.size());
  }
  build_nodes();
}

int Solver::node_for_level(int level) const {
  int best = -1;
  for (size_t i = 0; i < nodes.size(); ++i)
    if (nodes[i].level == level) best = (int)i;
  if (best < 0) throw tmg::Error("no such level");
  return best;
}

std::vector<NodeSpec> build_node_specs(const Owners& W, const ProblemDesc& prob, const MGDesc& mgd) {
  if (mgd.nlevels < 1) throw tmg::ConfigError("mg: number of levels must be >= 1");
  const int top = mgd.nlevels - 1;
  std::optional<std::array<int, 3>> hint;
  if (prob.pg_hint[0] || prob.pg_hint[1] || prob.pg_hint[2]) hint = prob.pg_hint;
  tmg::GridHeader H = tmg::build_header_for(W.R, 3, {prob.np[0], prob.np[1], prob.np[2]}, 1, 1, hint);
  std::vector<int> wr(W.R);
  for (int r = 0; r < W.R; ++r) wr[r] = r;

  auto tele = mgd.tele;
  std::sort(tele.begin(), tele.end(), [](const TeleStage& a, const TeleStage& b) { return a.level > b.level; });
  for (size_t t = 0; t < tele.size(); ++t) {
    if (tele[t].level < 0 || tele[t].level > top) throw tmg::ConfigError("telescope: level out of range");
    if (t && tele[t].level == tele[t - 1].level) throw tmg::ConfigError("telescope: two stages on one level");
    if (tele[t].r < 1) throw tmg::ConfigError("telescope: reduction factor must be >= 1");
  }
  std::vector<NodeSpec> out;
  const int T = (int)tele.size();
  int seg_top = top;
  for (int s = 0; s <= T; ++s) {
    const int bottom = s < T ? tele[s].level : 0;
    for (int l = seg_top; l >= bottom; --l) {
      NodeSpec nd;
      nd.level = l;
      nd.stage = (s < T && l == bottom) ? s : -1;
      nd.kind = (s < T && l == bottom) ? TELESCOPE : (l == 0 ? COARSE : SMOOTH);
      nd.dist = make_dist(W, H, wr);
      out.push_back(nd);
      if (l > bottom) {
        auto c = tmg::try_coarsen_header(H);
        if (!c)
          throw tmg::ConfigError("cannot coarsen: level " + std::to_string(l) + " grid " +
                                 std::to_string(H.npoints[0]) + "x" + std::to_string(H.npoints[1]) + "x" +
                                 std::to_string(H.npoints[2]) + " on a " + std::to_string(H.proc_grid[0]) + "x" +
                                 std::to_string(H.proc_grid[1]) + "x" + std::to_string(H.proc_grid[2]) +
                                 " processor grid (axes need 2M+1 vertices and every rank one vertex)");
        H = *c;
      }
    }
    if (s < T) {  // TelescopePC setup: split_strided + repartition_onto
      const tmg::SplitResult sp = tmg::split_strided(H.n_ranks(), tele[s].r);
      std::array<std::optional<int>, 3> ov;
      for (int a = 0; a < 3; ++a)
        if (tele[s].ov[a]) ov[a] = tele[s].ov[a];
      H = tmg::repartition_header(H, sp.n_members(), ov);
      std::vector<int> nwr;
      for (int mm : sp.member_map) nwr.push_back(wr[mm]);
      wr = nwr;
      seg_top = bottom;
    }
  }
  if (out.back().dist->h.n_ranks() != 1)
    throw tmg::ConfigError("pc_type lu needs a single-rank communicator; repartition first, e.g. pc_type telescope "
                           "with <prefix>telescope_pc_type lu");
  return out;
}

void Solver::build_nodes() {
  for (const NodeSpec& sp : build_node_specs(W, prob, mgd)) {
    Node nd;
    nd.kind = sp.kind;
    nd.level = sp.level;
    nd.stage = sp.stage;
    nd.dist = sp.dist;
    if (nd.kind == TELESCOPE) stage_node.push_back((int)nodes.size());
    nodes.push_back(std::move(nd));
  }

  // CG workspace; the top node's V-cycle input/output are the CG's r and z (fixed bindings,
  // so the captured iteration graph stays valid)
  {
    const Dist& D0 = *nodes[0].dist;
    cx = make_field(arena, D0);
    cr = make_field(arena, D0);
    cz = make_field(arena, D0);
    cp = make_field(arena, D0);
    cp2 = make_field(arena, D0);
    cw = make_field(arena, D0);
  }
  // buffers, operators, plans
  int nloc_max = 1;
  for (size_t ni = 0; ni < nodes.size(); ++ni) {
    Node& nd = nodes[ni];
    const Dist& D = *nd.dist;
    nloc_max = std::max<int>(nloc_max, (int)D.local.size());
    if (prob.kind == 1) {
      nd.kcoef = make_field(arena, D);
      for (size_t q = 0; q < D.local.size(); ++q)
        W.cnt.launches += launch_fill_coeff(D.geo[q], nd.kcoef.p[q], spheres_dev, (int)spheres.size(), prob.k_in,
                                            true, W.stream);
    }
    for (size_t q = 0; q < D.local.size(); ++q) {
      OpParams op = make_op(D.h);
      if (prob.kind == 1) {
        op.k = nd.kcoef.p[q];
        // precomputed rows (D, FX, FY, FZ) used by the stencil passes of this level
        double* fc = arena.alloc(4 * D.geo[q].total);
        W.cnt.launches += launch_fill_faces(D.geo[q], op, fc, D.geo[q].total, W.stream);
        op.fc = fc;
        op.fc_stride = D.geo[q].total;
      }
      nd.op.push_back(op);
      nblk_max = std::max(nblk_max, grid_blocks(D.geo[q]));
      staging_n = std::max<long long>(staging_n, D.local_unknowns());
    }
    nd.b = ni == 0 ? cr : make_field(arena, D);
    nd.x = ni == 0 ? cz : make_field(arena, D);
    if (nd.kind == SMOOTH) {
      nd.r = make_field(arena, D);
      nd.d = make_field(arena, D);
      nd.d2 = make_field(arena, D);
    }
    nd.halo = upload_plan(arena, halo_plan_host(W, D));
  }
  for (size_t i = 0; i < nodes.size(); ++i)
    if (nodes[i].kind == TELESCOPE) {  // TelescopePC setup: the P-hat^T / ScatterPlan data movement
      const auto t0 = std::chrono::steady_clock::now();
      nodes[i].gather = upload_plan(arena, transfer_plan_host(W, *nodes[i].dist, *nodes[i + 1].dist));
      nodes[i].scatter = upload_plan(arena, transfer_plan_host(W, *nodes[i + 1].dist, *nodes[i].dist));
      sync();
      nodes[i].t_setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
  part = arena.alloc((long long)nloc_max * 2 * nblk_max);
  for (int q = 0; q < nloc_max; ++q) part_off.push_back((long long)q * 2 * nblk_max);
  for (Node& nd : nodes) {  // creation order, identical on every process
    plans.push_back(&nd.halo);
    if (nd.kind == TELESCOPE) {
      plans.push_back(&nd.gather);
      plans.push_back(&nd.scatter);
    }
  }
  wire_transport();  // allocates rank_sums (+ the IPC mailbox when P > 1)
  scal = arena.alloc(S_NSLOTS);
  CK(cudaMallocHost(&host_scal, sizeof(double) * (S_NSLOTS + 2 * W.R + 8)));
  staging = arena.alloc(staging_n);
  {
    const Dist& D0 = *nodes[0].dist;
    ranks_dev = arena.alloc_t<int>(D0.h.n_ranks());
    arena.upload(ranks_dev, D0.wr.data(), sizeof(int) * D0.wr.size());
  }
  if (mgd.galerkin) build_galerkin();
  setup_coarse(nodes.back());
  sync();

  // Chebyshev intervals: given, or estimated (SolverNode::create, solver.cpp:591-592)
  for (size_t i = 0; i < nodes.size(); ++i) {
    Node& nd = nodes[i];
    if (nd.kind != SMOOTH) continue;
    if (!mgd.bounds.empty()) {
      nd.lo = mgd.bounds[2 * nd.level];
      nd.hi = mgd.bounds[2 * nd.level + 1];
    } else {
      estimate((int)i, mgd.est_mode);
    }
  }
  sync();
  cc_from = coarse_chain_start();
}

// Cross-process wiring (P > 1): one mailbox allocation per process holds the rank_sums slots
// and every plan's receive area; its CUDA IPC handle and the per-plan segment offsets are
// allgathered once, after which each pack descriptor points straight at its segment in the
// receiving process's mailbox. Single process: rank_sums only, no mailbox.
namespace {
struct Pub {
  cudaIpcMemHandle_t handle;
  int nplans;
};
void put(std::string& s, const void* p, size_t n) { s.append(static_cast<const char*>(p), n); }
template <class T>
T take(const std::string& s, size_t& at) {
  T v;
  std::memcpy(&v, s.data() + at, sizeof(T));
  at += sizeof(T);
  return v;
}
}  // namespace

void Solver::wire_transport() {
  if (W.P == 1) {
    rank_sums = arena.alloc(2LL * W.R);
    return;
  }
  mailbox = wire_plans(W, arena, plans, 2LL * W.R, peer_mail);
  rank_sums = mailbox;
}

double* wire_plans(World& W, DeviceArena& arena, const std::vector<RegionPlan*>& plans, long long head,
                   std::vector<double*>& peer_mail) {
  long long off = head;
  for (RegionPlan* p : plans) {
    p->mb_off = off;
    off += p->recv_total;
  }
  double* mailbox = arena.alloc(off);
  CK(cudaStreamSynchronize(W.stream));
  W.check();
  for (RegionPlan* p : plans) p->recvbuf = p->recv_total ? mailbox + p->mb_off : nullptr;
  // publication: handle, then per plan {send_total, nrecvs, (src proc, segment offset)...}
  std::string mine;
  Pub pub{};
  CK(cudaIpcGetMemHandle(&pub.handle, mailbox));
  pub.nplans = (int)plans.size();
  put(mine, &pub, sizeof pub);
  for (RegionPlan* p : plans) {
    const long long st = p->send_total;
    const int nr = (int)p->recvs.size();
    put(mine, &st, sizeof st);
    put(mine, &nr, sizeof nr);
    for (const auto& r : p->recvs) {
      const long long seg = p->mb_off + r.off;
      put(mine, &r.proc, sizeof r.proc);
      put(mine, &seg, sizeof seg);
    }
  }
  const std::vector<std::string> all = W.grp->allgather(mine);
  peer_mail.assign((size_t)W.P, nullptr);
  // seg[q][k][src] = offset of src's segment in q's mailbox for plan k
  std::vector<std::vector<std::vector<long long>>> seg((size_t)W.P);
  std::vector<char> xproc(plans.size(), 0);
  for (int q = 0; q < W.P; ++q) {
    size_t at = 0;
    const Pub pq = take<Pub>(all[(size_t)q], at);
    if (pq.nplans != (int)plans.size()) throw tmg::Error("transport: processes built different plan lists");
    seg[(size_t)q].assign(plans.size(), std::vector<long long>((size_t)W.P, -1));
    for (size_t k = 0; k < plans.size(); ++k) {
      const long long st = take<long long>(all[(size_t)q], at);
      const int nr = take<int>(all[(size_t)q], at);
      if (st > 0) xproc[k] = 1;
      for (int j = 0; j < nr; ++j) {
        const int src = take<int>(all[(size_t)q], at);
        seg[(size_t)q][k][(size_t)src] = take<long long>(all[(size_t)q], at);
      }
    }
    if (q != W.me) {
      void* ptr = nullptr;
      CK(cudaIpcOpenMemHandle(&ptr, pq.handle, cudaIpcMemLazyEnablePeerAccess));
      peer_mail[(size_t)q] = static_cast<double*>(ptr);
    }
  }
  for (size_t k = 0; k < plans.size(); ++k) {
    RegionPlan& p = *plans[k];
    p.xproc = xproc[k] != 0;
    if (!p.n_pack) continue;
    std::vector<long long> start((size_t)W.P, 0);
    for (const auto& sd : p.sends) start[(size_t)sd.proc] = sd.off;
    for (size_t d = 0; d < p.pack_h.size(); ++d) {
      const int q = p.pack_peer[d];
      const long long sg = seg[(size_t)q][k][(size_t)W.me];
      if (sg < 0) throw tmg::Error("transport: receiver has no segment for this sender");
      p.pack_h[d].dst_abs = peer_mail[(size_t)q] + sg;
      p.pack_h[d].dst_off -= start[(size_t)q];
    }
    arena.upload(p.d_pack, p.pack_h.data(), sizeof(CopyDesc) * p.pack_h.size());
  }
  W.grp->barrier();
  return mailbox;
}

// Galerkin coarse operators (mg_setup with galerkin; ptap dist_matrix.cpp:462-468):
// every level below the finest gets 27-point rows 2^-3 P^T A P computed on the device from the
// level above (whose 27 planes are halo-exchanged first). At a telescope stage the member
// operator is the parent's rows moved with the gather plan, i.e. C3(i) A' = P-hat^T A P-hat
// followed by row fusion, with no explicit permutation matrix.
void Solver::build_galerkin() {
  auto planes = [&](const Node& nd, int s) {
    Field f;
    for (size_t q = 0; q < nd.S.p.size(); ++q) f.p.push_back(nd.S.p[q] + (long long)s * nd.dist->geo[q].total);
    return f;
  };
  for (size_t i = 1; i < nodes.size(); ++i) {
    Node& nd = nodes[i];
    Node& up = nodes[i - 1];
    const Dist& D = *nd.dist;
    if (nd.level == up.level && up.S.p.empty()) continue;  // telescope of the finest (7-point) level
    for (const auto& g : D.geo) nd.S.p.push_back(arena.alloc(27 * g.total));
    if (nd.level == up.level) {
      for (int s = 0; s < 27; ++s) run_plan(W, up.gather, planes(up, s), planes(nd, s), true);
    } else {
      if (!up.S.p.empty())
        for (int s = 0; s < 27; ++s) run_plan(W, up.halo, planes(up, s), planes(up, s), false);
      for (size_t q = 0; q < D.local.size(); ++q)
        W.cnt.launches += launch_galerkin(up.dist->geo[q], up.op[q], D.geo[q], nd.S.p[q], D.geo[q].total,
                                          spheres_dev, (int)spheres.size(), prob.k_in, W.stream);
    }
    static const bool sym_env = [] {  // TMGX_G27_SYM=0: read all 27 planes in the perf build too
      const char* e = std::getenv("TMGX_G27_SYM");
      return e ? std::atoi(e) != 0 : true;
    }();
    for (size_t q = 0; q < D.local.size(); ++q) {
      const BoxGeo& g = D.geo[q];
      nd.op[q].S = nd.S.p[q];
      nd.op[q].S_stride = g.total;
      nd.op[q].sym27 = !parity_build() && sym_env && g.ex == g.Nx && g.ey == g.Ny && g.ez == g.Nz ? 1 : 0;
    }
  }
  sync();
}

// LUPC (precond.cpp:220-229): dense LU of the coarse operator, factored on the host with
// DenseLU::factor's partial pivoting (precond.cpp:11-48).
// DenseLU::factor (precond.cpp:11-48) of a dense row-major matrix and its device copy: the
// factors + pivots for the parity build's substitution (k_lu_solve), or the explicit inverse
// built from the same factors for the performance build (k_dense_matvec). map[c] = device
// offset of compact unknown c.
void dense_lu_setup(DeviceArena& arena, std::vector<double> a, int n, const std::vector<long long>& map,
                    double** A_dev, long long** piv_dev, long long** map_dev) {
  std::vector<long long> piv((size_t)n);
  for (int kk2 = 0; kk2 < n; ++kk2) {  // precond.cpp:26-46
    int p = kk2;
    double best = std::fabs(a[(size_t)kk2 * n + kk2]);
    for (int i = kk2 + 1; i < n; ++i)
      if (std::fabs(a[(size_t)i * n + kk2]) > best) {
        best = std::fabs(a[(size_t)i * n + kk2]);
        p = i;
      }
    if (best == 0.0) throw tmg::Error("lu factorization: matrix is singular at column " + std::to_string(kk2));
    piv[(size_t)kk2] = p;
    if (p != kk2)
      for (int j = 0; j < n; ++j) std::swap(a[(size_t)kk2 * n + j], a[(size_t)p * n + j]);
    const double pivot = a[(size_t)kk2 * n + kk2];
    for (int i = kk2 + 1; i < n; ++i) {
      const double m = a[(size_t)i * n + kk2] / pivot;
      a[(size_t)i * n + kk2] = m;
      if (m == 0.0) continue;
      for (int j = kk2 + 1; j < n; ++j) {
        volatile double t = m * a[(size_t)kk2 * n + j];
        a[(size_t)i * n + j] = a[(size_t)i * n + j] - t;
      }
    }
  }
  *map_dev = arena.alloc_t<long long>(n);
  arena.upload(*map_dev, map.data(), sizeof(long long) * n);
  *A_dev = arena.alloc((long long)n * n);
  if (parity_build()) {
    *piv_dev = arena.alloc_t<long long>(n);
    arena.upload(*piv_dev, piv.data(), sizeof(long long) * n);
    arena.upload(*A_dev, a.data(), sizeof(double) * (size_t)n * n);
  } else {
    // Performance build: explicit inverse from the same factors (columns = DenseLU::solve(e_c)),
    // applied as one warp-per-row matvec instead of a 2n-step dependent substitution chain.
    std::vector<double> inv((size_t)n * n), y((size_t)n), x((size_t)n);
    for (int c = 0; c < n; ++c) {
      std::fill(y.begin(), y.end(), 0.0);
      y[(size_t)c] = 1.0;
      for (int k = 0; k < n; ++k) {
        const long long p = piv[(size_t)k];
        if (p != k) std::swap(y[(size_t)k], y[(size_t)p]);
        for (int j = 0; j < k; ++j) y[(size_t)k] -= a[(size_t)k * n + j] * y[(size_t)j];
      }
      for (int k = n - 1; k >= 0; --k) {
        double acc = y[(size_t)k];
        for (int j = k + 1; j < n; ++j) acc -= a[(size_t)k * n + j] * x[(size_t)j];
        x[(size_t)k] = acc / a[(size_t)k * n + k];
      }
      for (int r = 0; r < n; ++r) inv[(size_t)r * n + c] = x[(size_t)r];
    }
    arena.upload(*A_dev, inv.data(), sizeof(double) * (size_t)n * n);
  }
}


void Solver::setup_coarse(Node& nd) {
  const Dist& D = *nd.dist;
  if (D.local.empty()) return;
  const BoxGeo& g = D.geo[0];
  const int nx = g.ex, ny = g.ey, nz = g.ez;
  const int n = nx * ny * nz;
  nd.nc = n;
  std::vector<double> a((size_t)n * n, 0.0);
  if (!nd.S.p.empty()) {  // 27-point Galerkin rows from the device
    std::vector<double> S((size_t)27 * g.total);
    CK(cudaMemcpyAsync(S.data(), nd.S.p[0], sizeof(double) * S.size(), cudaMemcpyDeviceToHost, W.stream));
    sync();
    for (int k = 0; k < nz; ++k)
      for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
          const int v = i + nx * (j + ny * k);
          const long long pv = g.base + i + g.px * j + g.pxy * k;
          for (int s = 0; s < 27; ++s) {
            const int dz = s / 9 - 1, dy = (s / 3) % 3 - 1, dx = s % 3 - 1;
            if (k + dz < 0 || k + dz >= nz || j + dy < 0 || j + dy >= ny || i + dx < 0 || i + dx >= nx) continue;
            a[(size_t)v * n + (v + dz * nx * ny + dy * nx + dx)] = S[(size_t)s * g.total + pv];
          }
        }
  }
  const OpParams op = make_op(D.h);
  std::vector<double> kk((size_t)n);
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) kk[(size_t)(i + nx * (j + ny * k))] = host_k(D, i, j, k);
  auto K = [&](int i, int j, int k) { return kk[(size_t)(i + nx * (j + ny * k))]; };
  for (int k = 0; k < nz && nd.S.p.empty(); ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const int v = i + nx * (j + ny * k);
        const bool bnd = i == 0 || j == 0 || k == 0 || i == nx - 1 || j == ny - 1 || k == nz - 1;
        const double kc = K(i, j, k);
        const double fzm = (k > 0 ? harm_h(kc, K(i, j, k - 1)) : kc) * op.ih2z;
        const double fym = (j > 0 ? harm_h(kc, K(i, j - 1, k)) : kc) * op.ih2y;
        const double fxm = (i > 0 ? harm_h(kc, K(i - 1, j, k)) : kc) * op.ih2x;
        const double fxp = (i + 1 < nx ? harm_h(kc, K(i + 1, j, k)) : kc) * op.ih2x;
        const double fyp = (j + 1 < ny ? harm_h(kc, K(i, j + 1, k)) : kc) * op.ih2y;
        const double fzp = (k + 1 < nz ? harm_h(kc, K(i, j, k + 1)) : kc) * op.ih2z;
        volatile double d = 0.0;
        d = d + fzm;
        d = d + fym;
        d = d + fxm;
        d = d + fxp;
        d = d + fyp;
        d = d + fzp;
        double* row = &a[(size_t)v * n];
        row[v] = d;
        if (bnd) continue;
        if (k - 1 > 0) row[v - nx * ny] = -fzm;
        if (j - 1 > 0) row[v - nx] = -fym;
        if (i - 1 > 0) row[v - 1] = -fxm;
        if (i + 1 < nx - 1) row[v + 1] = -fxp;
        if (j + 1 < ny - 1) row[v + nx] = -fyp;
        if (k + 1 < nz - 1) row[v + nx * ny] = -fzp;
      }
  std::vector<long long> map((size_t)n);
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) map[(size_t)(i + nx * (j + ny * k))] = g.base + i + g.px * j + g.pxy * k;
  dense_lu_setup(arena, a, n, map, &nd.A_dev, &nd.piv_dev, &nd.map_dev);
}

// ------------------------------------------------------------------------------------------
// primitives
// ------------------------------------------------------------------------------------------

void Solver::halo(int i, const Field& f) { run_plan(W, nodes[i].halo, f, f, false); }

void Solver::apply(int i, const Field& x, const Field& y) {
  Node& nd = nodes[i];
  halo(i, x);
  for (size_t q = 0; q < nd.dist->local.size(); ++q)
    W.cnt.launches += launch_apply(nd.dist->geo[q], nd.op[q], x.p[q], y.p[q], W.stream);
}

void Solver::coarse_solve(int i) {
  Node& nd = nodes[i];
  if (nd.dist->local.empty()) return;
  if (parity_build())
    W.cnt.launches += launch_lu_solve(nd.A_dev, nd.piv_dev, nd.nc, nd.map_dev, nd.b.p[0], nd.x.p[0], W.stream);
  else
    W.cnt.launches += launch_dense_matvec(nd.A_dev, nd.nc, nd.map_dev, nd.b.p[0], nd.x.p[0], W.stream);
}

// solve_fixed, Chebyshev branch (solver.cpp:79-110) fused into stencil passes:
//   pre (x = 0): d0 = D^-1 b / theta ; then m-1 passes  x += d ; r -= A d ; d = c1 d + c2 D^-1 r
//   post:        r = b - A x ; d0 = D^-1 r / theta ; then the same m-1 passes
// The last pass folds the final x += d and writes x only.
void Solver::smooth(int i, bool zero_x) {
  Node& nd = nodes[i];
  const Dist& D = *nd.dist;
  const int m = mgd.m;
  const double theta = 0.5 * (nd.hi + nd.lo);
  const double delta = 0.5 * (nd.hi - nd.lo);
  const double sigma = theta / delta;
  double rho = 1.0 / sigma;
  const double s_theta = 1.0 / theta;
  const size_t nb = D.local.size();
  if (use_tb(i)) {  // one temporally blocked kernel per side (bitwise identical arithmetic)
    if (!zero_x)  // the kernel reads x out of place
      for (size_t q = 0; q < nb; ++q) W.cnt.launches += launch_copy_interior(D.geo[q], nd.x.p[q], nd.d.p[q], W.stream);
    for (size_t q = 0; q < nb; ++q) tb_side(nd, q, nd.d.p[q], nd.x.p[q], zero_x);
    return;
  }
  if (zero_x) {
    for (size_t q = 0; q < nb; ++q)
      W.cnt.launches += launch_cheb_start_zero(D.geo[q], nd.op[q], nd.b.p[q], m == 1 ? nd.x.p[q] : nd.d.p[q], s_theta,
                                               W.stream);
    if (m == 1) return;
  } else {
    halo(i, nd.x);
    for (size_t q = 0; q < nb; ++q)
      W.cnt.launches += launch_cheb_start_res(D.geo[q], nd.op[q], nd.b.p[q], nd.x.p[q], nd.r.p[q], nd.d.p[q], s_theta,
                                              W.stream);
    if (m == 1) {
      for (size_t q = 0; q < nb; ++q) W.cnt.launches += launch_axpy(D.geo[q], 1.0, nd.d.p[q], nd.x.p[q], W.stream);
      return;
    }
  }
  for (int it = 0; it < m - 1; ++it) {
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    ChebStep cs{rho_new * rho, 2.0 * rho_new / delta};
    rho = rho_new;
    halo(i, nd.d);
    const bool first_zero = zero_x && it == 0;
    for (size_t q = 0; q < nb; ++q)
      W.cnt.launches += launch_cheb_step(D.geo[q], nd.op[q], nd.d.p[q], first_zero ? nd.b.p[q] : nd.r.p[q],
                                         first_zero ? nullptr : nd.x.p[q], nd.d2.p[q], nd.r.p[q], nd.x.p[q], cs,
                                         it == m - 2, W.stream);
    std::swap(nd.d, nd.d2);
  }
}

// First node of the trailing chain that the fused coarse V-cycle can run: single-box SMOOTH
// levels owned by this process, at most cc_max_extent vertices across (launch-latency bound),
// down to the COARSE (LU) node. -1: none (or TMGX_CC_MAX=0).
int Solver::coarse_chain_start() const {
  if (cc_max_extent <= 0 || nodes.empty() || nodes.back().kind != COARSE || nodes.back().dist->local.size() != 1 ||
      !coarse_cycle_supported(nodes.back().nc) || mgd.m - 1 > kCCMaxM)
    return -1;
  int i0 = -1;
  for (int i = (int)nodes.size() - 2; i >= 0; --i) {
    const Node& nd = nodes[i];
    const Dist& D = *nd.dist;
    if (nd.kind != SMOOTH || D.h.n_ranks() != 1 || D.local.size() != 1 || D.geo[0].ex > cc_max_extent ||
        D.geo[0].ey > cc_max_extent || D.geo[0].ez > cc_max_extent || (int)nodes.size() - 1 - i > kCCMaxLev)
      break;
    i0 = i;
  }
  return i0;
}

// The fused coarse V-cycle from node i0 (see tmgx_kernels.cuh): the same Chebyshev coefficients as
// smooth(), the nodes' b, x, r, d, d2 buffers, the coarse node's LU.
void Solver::coarse_cycle(int i0) {
  CCParams P{};
  P.m = mgd.m;
  P.nlev = (int)nodes.size() - 1 - i0;
  for (int l = 0; l <= P.nlev; ++l) {
    Node& nd = nodes[i0 + l];
    CCLevel& L = P.L[l];
    L.g = nd.dist->geo[0];
    L.b = nd.b.p[0];
    L.x = nd.x.p[0];
    if (nd.kind == COARSE) break;
    L.op = nd.op[0];
    L.r = nd.r.p[0];
    L.d = nd.d.p[0];
    L.d2 = nd.d2.p[0];
    const double theta = 0.5 * (nd.hi + nd.lo), delta = 0.5 * (nd.hi - nd.lo), sigma = theta / delta;
    L.s_theta = 1.0 / theta;
    double rho = 1.0 / sigma;
    for (int it = 0; it < mgd.m - 1; ++it) {
      const double rho_new = 1.0 / (2.0 * sigma - rho);
      L.cs[it] = ChebStep{rho_new * rho, 2.0 * rho_new / delta};
      rho = rho_new;
    }
  }
  const Node& cn = nodes.back();
  P.A = cn.A_dev;
  P.piv = cn.piv_dev;
  P.map = cn.map_dev;
  P.nc = cn.nc;
  W.cnt.launches += launch_coarse_cycle(P, W.stream);
}

// mg_apply (Alg. 1) over the node list; TELESCOPE nodes realise
// TelescopePC::apply: gather, inner V-cycle on the members, scatter back.
void Solver::vcycle(int i) {
  if (!prof) {
    vcycle_body(i);
    return;
  }
  LevelProf& P = (*prof)[(size_t)i];
  P.descended = false;
  P.recorded = true;
  P.bytes_in = W.cnt.halo_bytes + W.cnt.tele_bytes;
  cuda_check(cudaEventRecord(P.e[0], W.stream), "record");
  vcycle_body(i);
  cuda_check(cudaEventRecord(P.e[3], W.stream), "record");
  P.bytes_out = W.cnt.halo_bytes + W.cnt.tele_bytes;
}

// the coarser part of the cycle below node i (events around it when profiling)
void Solver::descend(int i) {
  if (!prof) {
    vcycle(i + 1);
    return;
  }
  LevelProf& P = (*prof)[(size_t)i];
  P.descended = true;
  P.bytes_down = W.cnt.halo_bytes + W.cnt.tele_bytes;
  cuda_check(cudaEventRecord(P.e[1], W.stream), "record");
  vcycle(i + 1);
  cuda_check(cudaEventRecord(P.e[2], W.stream), "record");
  P.bytes_up = W.cnt.halo_bytes + W.cnt.tele_bytes;
}

// Per-node exclusive device time and peer bytes of `reps` V-cycles (events on the library
// stream; the node's own kernels and exchanges, its coarser part excluded).
void Solver::level_profile(int reps, std::vector<double>& us, std::vector<long long>& bytes) {
  std::vector<LevelProf> lp(nodes.size());
  for (auto& P : lp)
    for (auto& e : P.e) cuda_check(cudaEventCreate(&e), "event");
  us.assign(nodes.size(), 0.0);
  bytes.assign(nodes.size(), 0);
  prof = &lp;
  try {
    for (int r = 0; r < reps; ++r) {
      for (auto& P : lp) P.recorded = false;
      vcycle(0);
      cuda_check(cudaStreamSynchronize(W.stream), "sync");
      for (size_t i = 0; i < nodes.size(); ++i) {
        LevelProf& P = lp[i];
        if (!P.recorded) continue;  // inside the fused coarse cycle: counted by its first node
        float a = 0.f, b = 0.f;
        if (P.descended) {
          cuda_check(cudaEventElapsedTime(&a, P.e[0], P.e[1]), "elapsed");
          cuda_check(cudaEventElapsedTime(&b, P.e[2], P.e[3]), "elapsed");
          bytes[i] += (P.bytes_down - P.bytes_in) + (P.bytes_out - P.bytes_up);
        } else {
          cuda_check(cudaEventElapsedTime(&a, P.e[0], P.e[3]), "elapsed");
          bytes[i] += P.bytes_out - P.bytes_in;
        }
        us[i] += 1e3 * (double)(a + b);
      }
    }
  } catch (...) {
    prof = nullptr;
    throw;
  }
  prof = nullptr;
  for (auto& P : lp)
    for (auto& e : P.e) cudaEventDestroy(e);
  for (size_t i = 0; i < nodes.size(); ++i) {
    us[i] /= reps;
    bytes[i] /= reps;
  }
}

void Solver::vcycle_body(int i) {
  Node& nd = nodes[i];
  if (i == 0) dots_nblk = 0;
  if (nd.kind == COARSE) {
    coarse_solve(i);
    return;
  }
  if (i == cc_from) {
    coarse_cycle(i);
    return;
  }
  if (nd.kind == TELESCOPE) {
    run_plan(W, nd.gather, nd.b, nodes[i + 1].b, true);
    descend(i);
    run_plan(W, nd.scatter, nodes[i + 1].x, nd.x, true);
    return;
  }
  const Dist& D = *nd.dist;
  Node& cn = nodes[i + 1];
  if (use_tb(i)) {
    // blocked pre-smooth b -> d (x after pre-smoothing), residual, restriction, coarse
    // correction x~ = d + P x_c into r (free after the restriction), blocked post-smooth r -> x
    for (size_t q = 0; q < D.local.size(); ++q) tb_side(nd, q, nullptr, nd.d.p[q], true);
    residual_restrict(i, nd.d);
    descend(i);
    halo(i + 1, cn.x);
    for (size_t q = 0; q < D.local.size(); ++q)
      W.cnt.launches += launch_prolong_to(D.geo[q], cn.dist->geo[q], cn.x.p[q], nd.d.p[q], nd.r.p[q], W.stream);
    if (i == 0 && D.local.size() == 1 && !parity_build() && fuse_dots)  // + the CG's r.z, z.z partials
      tb_side(nd, 0, nd.r.p[0], nd.x.p[0], false, true);
    else
      for (size_t q = 0; q < D.local.size(); ++q) tb_side(nd, q, nd.r.p[q], nd.x.p[q], false);
    return;
  }
  smooth(i, true);
  residual_restrict(i, nd.x);
  descend(i);
  halo(i + 1, cn.x);
  for (size_t q = 0; q < D.local.size(); ++q)
    W.cnt.launches += launch_prolong_add(D.geo[q], cn.dist->geo[q], cn.x.p[q], nd.x.p[q], W.stream);
  smooth(i, false);
}

// b_c = R (b - A x) of level i into the next node's b: fused on single-box 7-point levels
// (the residual stays on chip), else residual into r, box halo of r, restriction.
void Solver::residual_restrict(int i, const Field& x) {
  Node& nd = nodes[i];
  Node& cn = nodes[i + 1];
  const Dist& D = *nd.dist;
  if (!parity_build() && fuse_rr2 > 0 && D.h.n_ranks() == 1 && D.local.size() == 1 &&
      fuse_rr2 >= (nd.op[0].k != nullptr || nd.op[0].fc != nullptr ? 2 : 1) &&
      resid_restrict2_supported(D.geo[0], nd.op[0], cn.dist->geo[0])) {
    W.cnt.launches += launch_resid_restrict2(D.geo[0], nd.op[0], cn.dist->geo[0], nd.b.p[0], x.p[0], cn.b.p[0], W.stream);
    return;
  }
  if (D.h.n_ranks() == 1 && D.local.size() == 1 && resid_restrict_supported(nd.op[0]) && fuse_rr) {
    W.cnt.launches += launch_resid_restrict(D.geo[0], nd.op[0], cn.dist->geo[0], nd.b.p[0], x.p[0], cn.b.p[0], W.stream);
    return;
  }
  halo(i, x);
  for (size_t q = 0; q < D.local.size(); ++q)
    W.cnt.launches += launch_residual(D.geo[q], nd.op[q], nd.b.p[q], x.p[q], nd.r.p[q], W.stream);
  halo(i, nd.r);
  for (size_t q = 0; q < D.local.size(); ++q)
    W.cnt.launches += launch_restrict(D.geo[q], cn.dist->geo[q], nd.r.p[q], cn.b.p[q], W.stream);
}

// First Chebyshev step coefficients (solver.cpp:90-93, 106-108) for the m = 2 blocked kernel.
ChebStep Solver::cheb_first_step(const Node& nd) const {
  const double theta = 0.5 * (nd.hi + nd.lo);
  const double delta = 0.5 * (nd.hi - nd.lo);
  const double sigma = theta / delta;
  const double rho = 1.0 / sigma;
  const double rho_new = 1.0 / (2.0 * sigma - rho);
  return ChebStep{rho_new * rho, 2.0 * rho_new / delta};
}

// The temporally blocked smoothers (m = 2 and m = 3) run on single-box levels of 7-point
// operators (TMGX_TB=0 disables them).
bool Solver::use_tb(int i) const {
  const Node& nd = nodes[i];
  if (!tb_enabled || nd.kind != SMOOTH || nd.dist->h.n_ranks() != 1 || nd.dist->local.empty() ||
      nd.op[0].S != nullptr || nd.dist->geo[0].ex < tb_min_extent)
    return false;
  if (mgd.m == 2) return cheb2_tb_supported(nd.dist->geo[0]);
  if (mgd.m == 3) return tb3_enabled && cheb3_tb_supported(nd.dist->geo[0]);
  return false;
}

// One blocked smoother side on local box q: pre (x = 0): b -> xout; post: (b, xin) -> xout.
// dots: also the CG's r.z, z.z block partials (finest level, single box).
void Solver::tb_side(Node& nd, size_t q, const double* xin, double* xout, bool pre, bool dots) {
  const Dist& D = *nd.dist;
  const double s_theta = 1.0 / (0.5 * (nd.hi + nd.lo));
  const ChebStep cs = cheb_first_step(nd);
  double* dp = dots ? part + part_off[0] : nullptr;
  const int dmax = dots ? nblk_max : 0;
  int* nbp = dots ? &dots_nblk : nullptr;
  if (mgd.m == 2) {
    W.cnt.launches += launch_cheb2_tb(D.geo[q], nd.op[q], nd.b.p[q], xin, xout, s_theta, cs, pre, W.stream, dp,
                                      nblk_max, dmax, nbp);
    return;
  }
  // second step (solver.cpp:100-108 recurrence)
  const double theta = 0.5 * (nd.hi + nd.lo), delta = 0.5 * (nd.hi - nd.lo), sigma = theta / delta;
  const double rho1 = 1.0 / (2.0 * sigma - 1.0 / sigma);
  const double rho2 = 1.0 / (2.0 * sigma - rho1);
  const ChebStep cs2{rho2 * rho1, 2.0 * rho2 / delta};
  W.cnt.launches += launch_cheb3_tb(D.geo[q], nd.op[q], nd.b.p[q], xin, xout, s_theta, cs, cs2, pre, W.stream, dp,
                                    nblk_max, dmax, nbp);
}

// Cross-process scalar reduction: every process stores its rank slots into every peer's
// rank_sums, then one stream barrier; each process then sums the slots in rank order itself
// (identical on all processes, and identical to the single-process sum).
void Solver::device_allreduce_ranksums(int nslots) { push_ranksums(W, rank_sums, nslots, peer_mail, rs_last_bar); }

void push_ranksums(World& W, double* rank_sums, int nslots, const std::vector<double*>& peer_mail, long long& last_bar) {
  if (W.P == 1) return;
  if (last_bar == W.nbar) W.stream_barrier();  // peers done reading the previous values
  PtrTable peers{};
  int np = 0;
  for (int q = 0; q < W.P; ++q)
    if (q != W.me) peers.p[np++] = peer_mail[(size_t)q];
  W.cnt.launches += launch_push_ranksums(rank_sums, W.R, nslots, W.first, W.end, peers, np, W.stream);
  W.stream_barrier();
  last_bar = W.nbar;
  W.cnt.allreduces++;
}

// Single process: clear the slots (only the listed ranks' slots are ever summed). With peers
// storing into this buffer concurrently, clearing would race; every summed slot is rewritten.
void Solver::sync() {
  CK(cudaStreamSynchronize(W.stream));
  W.check();
}

void Solver::zero_ranksums() {
  if (W.P == 1) CK(cudaMemsetAsync(rank_sums, 0, sizeof(double) * 2 * W.R, W.stream));
}

// Deterministic collective sums for node i's distribution: per-box block partials are reduced
// in a fixed tree, then summed over the communicator's ranks in rank order (the reference's
// ordered_fold_sum, comm.cpp:338-351, at box granularity). Identical on every process.
// The parity build replaces the tree by the reference's serial left fold (a.b recomputed).
void Solver::reduce_local(const Dist& D, int nslots, const Field* a, const Field* b, const Field* c, int nblk) {
  for (size_t q = 0; q < D.local.size(); ++q) {
    double* out = rank_sums + D.wr[D.local[q]];
    if (parity_build() && a && b)
      W.cnt.launches += launch_fold_dot(D.geo[q], a->p[q], b->p[q], c ? c->p[q] : nullptr, out, W.R, W.stream);
    else
      W.cnt.launches += launch_reduce_partials(part + part_off[q], nblk > 0 ? nblk : grid_blocks(D.geo[q]), nslots,
                                               nblk_max, out, W.R, W.stream);
  }
}

std::array<double, 2> Solver::collect2(int i, int nslots, const Field* a, const Field* b) {
  const Dist& D = *nodes[i].dist;
  zero_ranksums();
  reduce_local(D, nslots, a, b, nullptr);
  device_allreduce_ranksums(nslots);
  CK(cudaMemcpyAsync(host_scal, rank_sums, sizeof(double) * 2 * W.R, cudaMemcpyDeviceToHost, W.stream));
  sync();
  std::array<double, 2> s{0.0, 0.0};
  for (int m = 0; m < D.h.n_ranks(); ++m) {
    s[0] += host_scal[D.wr[m]];
    s[1] += host_scal[W.R + D.wr[m]];
  }
  return s;
}

double tridiag_eig_max(const std::vector<double>& d, const std::vector<double>& e) {
  // solver.cpp:488-516 (Sturm bisection)
  const size_t n = d.size();
  double lo = d[0], hi = d[0];
  for (size_t i = 0; i < n; ++i) {
    const double left = i > 0 ? std::abs(e[i - 1]) : 0.0;
    const double right = i + 1 < n ? std::abs(e[i]) : 0.0;
    lo = std::min(lo, d[i] - left - right);
    hi = std::max(hi, d[i] + left + right);
  }
  auto count_below = [&](double x) {
    int count = 0;
    double q = 1.0;
    for (size_t i = 0; i < n; ++i) {
      const double off = i > 0 ? e[i - 1] : 0.0;
      q = d[i] - x - (q == 0.0 ? std::abs(off) / 1e-300 : off * off / q);
      if (q < 0.0) ++count;
    }
    return count;
  };
  for (int it = 0; it < 200 && hi - lo > 1e-12 * std::max(1.0, std::abs(hi)); ++it) {
    const double mid = 0.5 * (lo + hi);
    if (count_below(mid) >= (int)n)
      hi = mid;
    else
      lo = mid;
  }
  return 0.5 * (lo + hi);
}

// chebyshev_bounds_estimate (solver.cpp:520-581): ten Jacobi-preconditioned CG steps from
// fill_random(0x5eedbeef) keyed by natural index (SURVEY finding 4(b)). mode 0 reproduces the
// shipped loop (p never updated, solver.cpp:537-561); mode 1 adds p = z + beta p.
void Solver::estimate(int i, int mode) {
  Node& nd = nodes[i];
  const Dist& D = *nd.dist;
  const size_t nb = D.local.size();
  Field &r = nd.r, &z = nd.d, &p = nd.d2, &w = nd.x;
  for (size_t q = 0; q < nb; ++q) W.cnt.launches += launch_fill_rhs(D.geo[q], r.p[q], 0x5eedbeefULL, false, W.stream);
  for (size_t q = 0; q < nb; ++q)
    W.cnt.launches += launch_jacobi_dot(D.geo[q], nd.op[q], r.p[q], z.p[q], part + part_off[q], W.stream);
  double rz = collect2(i, 1, &r, &z)[0];
  for (size_t q = 0; q < nb; ++q) W.cnt.launches += launch_copy_interior(D.geo[q], z.p[q], p.p[q], W.stream);
  std::vector<double> alphas, betas;
  bool broke = false;
  for (int it = 0; it < 10; ++it) {
    if (rz == 0.0 || !std::isfinite(rz)) break;
    halo(i, p);
    for (size_t q = 0; q < nb; ++q)
      W.cnt.launches += launch_spmv_dot(D.geo[q], nd.op[q], p.p[q], w.p[q], part + part_off[q], W.stream);
    const double pw = collect2(i, 1, &p, &w)[0];
    if (pw <= 0.0 || !std::isfinite(pw)) {
      if (alphas.empty()) broke = true;
      break;
    }
    const double alpha = rz / pw;
    for (size_t q = 0; q < nb; ++q) W.cnt.launches += launch_axpy(D.geo[q], -alpha, w.p[q], r.p[q], W.stream);
    for (size_t q = 0; q < nb; ++q)
      W.cnt.launches += launch_jacobi_dot(D.geo[q], nd.op[q], r.p[q], z.p[q], part + part_off[q], W.stream);
    const double rz_new = collect2(i, 1, &r, &z)[0];
    alphas.push_back(alpha);
    if (rz_new <= 0.0 || !std::isfinite(rz_new)) break;
    const double beta = rz_new / rz;
    betas.push_back(beta);
    rz = rz_new;
    if (mode == 1) {
      double* hb = host_scal + S_NSLOTS + 2 * W.R;
      *hb = beta;
      CK(cudaMemcpyAsync(scal + S_TMP0, hb, sizeof(double), cudaMemcpyHostToDevice, W.stream));
      for (size_t q = 0; q < nb; ++q) W.cnt.launches += launch_p_update(D.geo[q], z.p[q], p.p[q], scal, S_TMP0, W.stream);
      sync();
    }
  }
  if (broke || alphas.empty()) {
    nd.lo = 0.1;
    nd.hi = 1.1;
    return;
  }
  const size_t k = alphas.size();
  std::vector<double> d(k, 0.0), e(k > 0 ? k - 1 : 0, 0.0);
  for (size_t t = 0; t < k; ++t) {
    d[t] = 1.0 / alphas[t];
    if (t > 0) d[t] += betas[t - 1] / alphas[t - 1];
    if (t + 1 < k) e[t] = std::sqrt(betas[t]) / alphas[t];
  }
  const double lam = tridiag_eig_max(d, e);
  if (!(lam > 0.0) || !std::isfinite(lam)) {
    nd.lo = 0.1;
    nd.hi = 1.1;
    return;
  }
  nd.lo = 0.1 * lam;
  nd.hi = 1.1 * lam;
}

void Solver::upload(int i, const Field& f, const double* src, bool on_device) {
  const Dist& D = *nodes[i].dist;
  long long off = 0;
  for (size_t q = 0; q < D.local.size(); ++q) {
    const BoxGeo& g = D.geo[q];
    const long long n = (long long)g.ex * g.ey * g.ez;
    const double* s = src + off;
    if (!on_device) {
      CK(cudaMemcpyAsync(staging, s, sizeof(double) * n, cudaMemcpyHostToDevice, W.stream));
      s = staging;
    }
    W.cnt.launches += launch_compact_to_box(g, s, f.p[q], W.stream);
    if (!on_device) sync();
    off += n;
  }
}

void Solver::download(int i, const Field& f, double* dst, bool on_device) {
  const Dist& D = *nodes[i].dist;
  long long off = 0;
  for (size_t q = 0; q < D.local.size(); ++q) {
    const BoxGeo& g = D.geo[q];
    const long long n = (long long)g.ex * g.ey * g.ez;
    if (on_device) {
      W.cnt.launches += launch_box_to_compact(g, f.p[q], dst + off, W.stream);
    } else {
      W.cnt.launches += launch_box_to_compact(g, f.p[q], staging, W.stream);
      CK(cudaMemcpyAsync(dst + off, staging, sizeof(double) * n, cudaMemcpyDeviceToHost, W.stream));
      sync();
    }
    off += n;
  }
}

// krylov_solve -> solve_cg (solver.cpp:214-266) with PcApply = one V-cycle. Scalars stay on
// the device; one CG iteration (p = z + beta p, w = A p with p.w, x/r update, V-cycle, r.z and
// z.z) is a single CUDA-graph launch, after which the host reads {pw, ||z||, flags} for the
// stopping test ||z_k|| <= max(rtol ||z_0||, atol) (solver.cpp:71-77).
void Solver::cg_dots(int op) {
  const Dist& D = *nodes[0].dist;
  zero_ranksums();
  const int fused = parity_build() ? 0 : dots_nblk;  // r.z, z.z partials from the finest post-smooth
  if (!parity_build() && !fused)
    for (size_t q = 0; q < D.local.size(); ++q)
      W.cnt.launches += launch_dot2(D.geo[q], cr.p[q], cz.p[q], cz.p[q], part + part_off[q],
                                    part + part_off[q] + nblk_max, W.stream);
  reduce_local(D, 2, &cr, &cz, &cz, fused);
  device_allreduce_ranksums(2);
  W.cnt.launches += launch_cg_scalars(op, rank_sums, W.R, ranks_dev, D.h.n_ranks(), scal, W.stream);
}

// Single-box fine level: p = z + beta p fused into w = A p (ping-pong between cp and cp2 by
// iteration parity, one captured graph per parity).
bool Solver::fused_cg() const {
  const Node& top = nodes[0];
  return fuse_cg && top.dist->h.n_ranks() == 1 && top.dist->local.size() == 1 && pspmv_supported(top.op[0]);
}

void Solver::cg_iteration(int par) {
  Node& top = nodes[0];
  const Dist& D = *top.dist;
  const size_t nb = D.local.size();
  const bool fused = fused_cg();
  Field& pn = (fused && par == 0) ? cp2 : cp;  // direction written this iteration
  zero_ranksums();
  if (fused) {
    const Field& po = par == 0 ? cp : cp2;
    W.cnt.launches += launch_pspmv_dot(D.geo[0], top.op[0], cz.p[0], po.p[0], pn.p[0], cw.p[0], part + part_off[0],
                                       scal, S_BETA, W.stream);
  } else {
    for (size_t q = 0; q < nb; ++q)
      W.cnt.launches += launch_p_update(D.geo[q], cz.p[q], cp.p[q], scal, S_BETA, W.stream);
    halo(0, cp);
    for (size_t q = 0; q < nb; ++q)
      W.cnt.launches += launch_spmv_dot(D.geo[q], top.op[q], cp.p[q], cw.p[q], part + part_off[q], W.stream);
  }
  reduce_local(D, 1, &pn, &cw, nullptr);
  device_allreduce_ranksums(1);
  W.cnt.launches += launch_cg_scalars(CG_ALPHA, rank_sums, W.R, ranks_dev, D.h.n_ranks(), scal, W.stream);
  for (size_t q = 0; q < nb; ++q)
    W.cnt.launches += launch_cg_update(D.geo[q], pn.p[q], cw.p[q], cx.p[q], cr.p[q], scal, S_ALPHA, S_FLAG_PW,
                                       W.stream);
  vcycle(0);
  cg_dots(CG_BETA);
  CK(cudaMemcpyAsync(host_scal, scal, sizeof(double) * S_NSLOTS, cudaMemcpyDeviceToHost, W.stream));
}

void Solver::run_iteration(int par) {
  if (!fused_cg()) par = 0;
  if (!use_graphs) {
    cg_iteration(par);
    return;
  }
  if (!iter_exec[par]) {
    const long long l0 = W.cnt.launches, b0 = W.nbar;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(W.stream, cudaStreamCaptureModeThreadLocal));
    cg_iteration(par);
    CK(cudaStreamEndCapture(W.stream, &g));
    CK(cudaGraphInstantiate(&iter_exec[par], g, 0));
    CK(cudaGraphDestroy(g));
    iter_launches = W.cnt.launches - l0;
    iter_bars = W.nbar - b0;  // stream barriers (host nodes) in one iteration
    W.cnt.launches = l0;
    W.nbar = b0;
    graph_base = b0;
  }
  // Host barrier bookkeeping of a replay: the plans used in the graph last published at
  // (previous start + their offset inside the iteration); move them to this replay's start.
  const long long shift = W.nbar - graph_base;
  if (shift) {
    for (RegionPlan* p : plans)
      if (p->last_bar > graph_base) p->last_bar += shift;
    if (rs_last_bar > graph_base) rs_last_bar += shift;
  }
  graph_base = W.nbar;
  CK(cudaGraphLaunch(iter_exec[par], W.stream));
  W.cnt.launches += iter_launches;
  W.nbar += iter_bars;
}

// Device inputs (tmgx.h stream contract): the library's stream waits for all work submitted so far
// to the legacy default stream (torch's default stream), so a caller that filled b / x there
// needs no extra synchronisation. Work on other caller streams must be synchronised by the caller.
void Solver::order_after_caller() {
  if (!caller_ev) CK(cudaEventCreateWithFlags(&caller_ev, cudaEventDisableTiming));
  CK(cudaEventRecord(caller_ev, cudaStreamLegacy));
  CK(cudaStreamWaitEvent(W.stream, caller_ev, 0));
}

Solver::~Solver() {
  if (W.grp) {  // collective teardown: no peer may still store into our mailbox
    cudaStreamSynchronize(W.stream);
    try {
      W.grp->barrier(30.0);
    } catch (...) {
    }
    for (double* p : peer_mail)
      if (p) cudaIpcCloseMemHandle(p);
  }
  if (caller_ev) cudaEventDestroy(caller_ev);
  for (auto& e : iter_exec)
    if (e) cudaGraphExecDestroy(e);
  if (host_scal) cudaFreeHost(host_scal);
}

int Solver::solve(const double* b, double* x, bool on_device, int method, double rtol, double atol, int max_its,
                  double* hist, int* reason, int* its, double* norm0, double* normf, double* t_ms, bool seeded,
                  unsigned long long seed, bool x0_nonzero) {
  CK(cudaSetDevice(W.device));
  Node& top = nodes[0];
  const Dist& D = *top.dist;
  const size_t nb = D.local.size();
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  if (on_device) order_after_caller();
  CK(cudaEventRecord(e0, W.stream));
  *its = 0;
  *reason = 2;  // max_its
  // b -> cw (temporary), x0 -> cx. With a zero initial guess r0 = b - A 0 = b bit for bit (every
  // row sum is +0), so b goes straight into r and the residual pass is skipped.
  const bool x0_zero = method != 5 && !(x && !seeded && x0_nonzero);
  Field& bdst = x0_zero ? cr : cw;
  if (seeded) {
    for (size_t q = 0; q < nb; ++q) W.cnt.launches += launch_fill_rhs(D.geo[q], bdst.p[q], seed, true, W.stream);
  } else {
    upload(0, bdst, b, on_device);
  }
  int rc = 0;
  if (method == 5) {  // preonly: x = M b
    for (size_t q = 0; q < nb; ++q) W.cnt.launches += launch_copy_interior(D.geo[q], cw.p[q], cr.p[q], W.stream);
    vcycle(0);
    if (x) download(0, cz, x, on_device);
    *reason = 3;
    *its = 1;
    *norm0 = *normf = 0.0;
  } else {
    if (!x0_zero) {
      upload(0, cx, x, on_device);
      halo(0, cx);
      for (size_t q = 0; q < nb; ++q)
        W.cnt.launches += launch_residual(D.geo[q], top.op[q], cw.p[q], cx.p[q], cr.p[q], W.stream);
    } else {
      for (size_t q = 0; q < nb; ++q) CK(cudaMemsetAsync(cx.p[q], 0, sizeof(double) * D.geo[q].total, W.stream));
    }
    vcycle(0);
    cg_dots(CG_INIT);  // also sets beta = 0 so that the first p = z + 0 p = z
    CK(cudaMemcpyAsync(host_scal, scal, sizeof(double) * S_NSLOTS, cudaMemcpyDeviceToHost, W.stream));
    sync();
    const double nrm0 = host_scal[S_NRM];
    *norm0 = nrm0;
    *normf = nrm0;
    if (hist) hist[0] = nrm0;
    const double tol = std::max(rtol * nrm0, atol);
    if (nrm0 <= tol) {
      *reason = nrm0 <= atol ? 1 : 0;
    } else {
      for (size_t q = 0; q < nb; ++q) {
        CK(cudaMemsetAsync(cp.p[q], 0, sizeof(double) * D.geo[q].total, W.stream));
        CK(cudaMemsetAsync(cp2.p[q], 0, sizeof(double) * D.geo[q].total, W.stream));
      }
      for (int it = 1; it <= max_its; ++it) {
        run_iteration((it - 1) & 1);
        sync();
        if (host_scal[S_FLAG_PW] != 0.0) {  // solver.cpp:237-241 (x, r not updated)
          *reason = 4;
          rc = 2;
          break;
        }
        const double nrm = host_scal[S_NRM];
        *its = it;
        *normf = nrm;
        if (hist) hist[it] = nrm;
        if (nrm <= tol) {
          *reason = nrm <= atol ? 1 : 0;
          break;
        }
        if (host_scal[S_FLAG_RZ] != 0.0) {  // solver.cpp:254-258
          *reason = 4;
          rc = 2;
          break;
        }
      }
    }
    if (x) download(0, cx, x, on_device);
  }
  CK(cudaEventRecord(e1, W.stream));
  CK(cudaEventSynchronize(e1));
  W.check();
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *t_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CK(cudaGetLastError());
  return rc;
}

}  // namespace tmgx
