// Host orchestration of the B200 MG-CG path: worlds, box distributions, halo and telescope
// plans, the MG node list, the Chebyshev interval estimator and the CG loop.
//
// Reference correspondence:
//   World            spawn_world / Comm (comm.hpp:75-207): R reference ranks over P processes
//   Dist             StructuredGrid (grid.hpp:85-118) bound to a (sub-)communicator
//   RegionPlan       ghost_exchange (grid.cpp:645-696) and ScatterPlan::to_sub/from_sub composed
//                    with P-hat (scatter_plan.cpp:40-114, grid.cpp:582-599)
//   MG nodes         mg_setup / mg_apply (missing mg.cpp) with
//                    TelescopePC (missing telescope.cpp) and LUPC (precond.cpp:220-229)
//   estimate_bounds  chebyshev_bounds_estimate (solver.cpp:520-581)
//   solve_cg         solve_cg (solver.cpp:214-266)
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "tmg_grid.hpp"
#include "tmgx_kernels.cuh"
#include "tmgx_node.hpp"

namespace tmgx {

void cuda_check(cudaError_t e, const char* what);

struct Counters {
  long long launches = 0;
  long long halo_bytes = 0;
  long long tele_bytes = 0;
  long long allreduces = 0;
};

// Which process owns which reference rank: process p owns [p*R/P, (p+1)*R/P).
struct Owners {
  int R = 1;  // reference ranks (grid boxes)
  int P = 1, me = 0;
  int first = 0, end = 1;  // local reference ranks
  Owners() = default;
  Owners(int R, int P, int me);
  int owner(int world_rank) const;
  bool local(int world_rank) const { return owner(world_rank) == me; }
};

// R reference ranks over P processes (one GPU each in production; any number sharing a GPU in
// tests). Processes synchronise only through stream-ordered host barriers (NodeGroup).
struct World : Owners {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::unique_ptr<NodeGroup> grp;  // P > 1
  long long nbar = 0;              // stream barriers enqueued so far (identical on every process)
  Counters cnt;

  World(int R, int P, int me, int device, const char* job);
  ~World();
  void stream_barrier();  // every process's stream reaches this point before any proceeds
  void check() const;     // throws if a stream barrier failed (timeout / peer abort)
};

// A GridHeader over a communicator whose comm rank m is reference rank wr[m].
struct Dist {
  tmg::GridHeader h;
  std::vector<int> wr;
  std::vector<int> local;  // comm ranks owned here, ascending
  std::vector<BoxGeo> geo;  // aligned with local
  int slot_of(int m) const;
  long long local_unknowns() const;
};

std::shared_ptr<Dist> make_dist(const Owners& W, const tmg::GridHeader& h, const std::vector<int>& wr);

// Per-local-box device buffers of one logical vector.
struct Field {
  std::vector<double*> p;
  PtrTable table() const;
};

// Device allocations of one solver. Every buffer is zeroed, and every host upload is issued, in
// stream order on the owner's stream (cudaStreamNonBlocking streams do not order against the
// legacy default stream, so a plain cudaMemset/cudaMemcpy could land after the setup kernels that
// follow it on that stream).
class DeviceArena {
 public:
  ~DeviceArena();
  void set_stream(cudaStream_t s) { stream_ = s; }
  double* alloc(long long n);
  template <class T>
  T* alloc_t(long long n) {
    return reinterpret_cast<T*>(alloc((n * (long long)sizeof(T) + 7) / 8));
  }
  // H2D copy on the arena's stream; returns when the copy is complete (src may be a temporary)
  void upload(void* dst, const void* src, size_t bytes);

 private:
  std::vector<void*> ptrs_;
  cudaStream_t stream_ = nullptr;
};

Field make_field(DeviceArena& A, const Dist& D);
double hashed_uniform_h(unsigned long long seed, unsigned long long idx);  // common.hpp:50-53
double tridiag_eig_max(const std::vector<double>& d, const std::vector<double>& e);  // solver.cpp:488-516
void dense_lu_setup(DeviceArena& arena, std::vector<double> a, int n, const std::vector<long long>& map,
                    double** A_dev, long long** piv_dev, long long** map_dev);

// Region copies between two distributions (halo: same dist, box halo incl. corners).
// Cross-process movement: the pack kernel stores each region straight into the receiving
// process's mailbox (peer pointer from its CUDA IPC handle), a stream barrier publishes it, and
// the receiver unpacks from its own mailbox. Same-process regions are one copy kernel.
struct RegionPlan {
  CopyDesc* d_local = nullptr;
  int n_local = 0, max_local = 0;
  CopyDesc* d_pack = nullptr;
  int n_pack = 0, max_pack = 0;
  CopyDesc* d_unpack = nullptr;
  int n_unpack = 0, max_unpack = 0;
  struct Peer {
    int proc;
    long long off, count;
  };
  std::vector<Peer> sends, recvs;
  long long send_total = 0, recv_total = 0;
  double* recvbuf = nullptr;      // this process's mailbox area of the plan
  long long mb_off = 0;           // its offset in the mailbox
  std::vector<CopyDesc> pack_h;   // host copies of the pack descriptors (rewired to peer pointers)
  std::vector<int> pack_peer;     // destination process of each pack descriptor
  bool xproc = false;             // some process pair exchanges data (global, same on all)
  long long last_bar = -1;        // W.nbar right after the last use's publishing barrier
  bool empty() const { return n_local == 0 && sends.empty() && recvs.empty(); }
};

// Host half of a plan: descriptors in (target rank asc, source rank asc) order, identical on
// both ends of every process pair; per-peer segment sizes and a checksum of the global vertex
// indices moved (for cross-process consistency tests).
struct PlanHost {
  std::vector<CopyDesc> loc, pack, unpack;
  std::vector<RegionPlan::Peer> sends, recvs;
  std::vector<unsigned long long> send_sum, recv_sum;  // aligned with sends / recvs
  std::vector<int> pack_peer;                          // destination process of each pack descriptor
  long long local_count = 0;
  int max_local = 0, max_pack = 0, max_unpack = 0;
  long long send_total = 0, recv_total = 0;
};
PlanHost halo_plan_host(const Owners& W, const Dist& D);
PlanHost transfer_plan_host(const Owners& W, const Dist& S, const Dist& T);
// the same plan for `ncomp` consecutive component planes per box (one barrier for all of them)
PlanHost expand_components(const PlanHost& h, const Dist& S, const Dist& T, int ncomp);
RegionPlan upload_plan(DeviceArena& A, const PlanHost& h);
void run_plan(World& W, RegionPlan& plan, const Field& src, const Field& dst, bool telescope);
// Cross-process wiring (P > 1): one CUDA-IPC mailbox per process holding `head` doubles (the
// rank-sum slots) followed by every plan's receive area; pack descriptors are rewired to the
// peers' mailboxes. Collective; returns this process's mailbox.
double* wire_plans(World& W, DeviceArena& A, const std::vector<RegionPlan*>& plans, long long head,
                   std::vector<double*>& peer_mail);
// Rank-ordered allreduce of [2][R] rank-sum slots: this process's slots stored into every peer's
// mailbox head, then a stream barrier (no-op when P == 1).
void push_ranksums(World& W, double* rank_sums, int nslots, const std::vector<double*>& peer_mail, long long& last_bar);

struct ProblemDesc {
  int kind = 0;  // 0 POISSON7, 1 VARCOEF7_HARMONIC
  std::array<long long, 3> np{65, 65, 65};
  std::array<int, 3> pg_hint{0, 0, 0};
  unsigned long long seed_k = 7;
  int n_spheres = 32;
  double k_in = 1e4;
};

struct TeleStage {
  int level;
  int r;
  std::array<int, 3> ov;
};

struct MGDesc {
  int nlevels = 5;
  int m = 2;
  int est_mode = 1;  // 0 reference, 1 lanczos
  std::vector<double> bounds;  // optional 2*nlevels
  std::vector<TeleStage> tele;
  bool galerkin = false;  // levels below the finest: 2^-3 P^T A P (27-point)
};

enum NodeKind { SMOOTH = 0, TELESCOPE = 1, COARSE = 2 };

// The V-cycle node list (host-only): outer levels on the world, TELESCOPE nodes at each stage
// level, the members' inner levels, COARSE (LU) at level 0 on a single rank.
struct NodeSpec {
  NodeKind kind;
  int level;
  int stage;
  std::shared_ptr<Dist> dist;
};
std::vector<NodeSpec> build_node_specs(const Owners& W, const ProblemDesc& P, const MGDesc& M);

struct Node {
  NodeKind kind;
  int level;
  int stage;  // telescope stage index for TELESCOPE nodes
  std::shared_ptr<Dist> dist;
  std::vector<OpParams> op;  // per local box
  Field kcoef, b, x, r, d, d2;
  Field S;  // Galerkin: per box 27 planes of `total` doubles (empty: 7-point operator)
  RegionPlan halo;
  double lo = 0.1, hi = 1.1;
  // telescope
  RegionPlan gather, scatter;
  double t_setup_s = 0.0;  // host time of the stage's plan construction + upload
  // coarse
  int nc = 0;
  double* A_dev = nullptr;  // Ainv (perf) or LU (parity)
  long long* piv_dev = nullptr;
  long long* map_dev = nullptr;
};

class Solver {
 public:
  Solver(World& W, const ProblemDesc& P, const MGDesc& M);
  ~Solver();
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;

  World& W;
  ProblemDesc prob;
  MGDesc mgd;
  DeviceArena arena;
  std::vector<Node> nodes;
  std::vector<int> stage_node;  // node index of each TELESCOPE node
  Sphere* spheres_dev = nullptr;
  std::vector<Sphere> spheres;

  // CG workspace on the top node's distribution
  Field cx, cr, cz, cp, cp2, cw;
  double* part = nullptr;       // per local box partials [box][2][nblk]
  std::vector<long long> part_off;
  int nblk_max = 0;
  double* rank_sums = nullptr;  // [2][R]; P > 1: the head of this process's IPC mailbox
  double* mailbox = nullptr;
  std::vector<double*> peer_mail;  // peers' mailboxes (IPC-mapped), nullptr for this process
  long long rs_last_bar = -1;
  std::vector<RegionPlan*> plans;  // every plan in creation order (identical on all processes)
  void wire_transport();
  double* scal = nullptr;       // S_NSLOTS
  double* host_scal = nullptr;  // pinned
  int* ranks_dev = nullptr;     // comm ranks -> world ranks of the top dist
  double* staging = nullptr;    // compact I/O staging (device)
  long long staging_n = 0;

  int node_for_level(int level) const;
  long long local_n(int node) const { return nodes[node].dist->local_unknowns(); }

  // primitives
  void vcycle(int i);  // nodes[i].b -> nodes[i].x
  void vcycle_body(int i);
  void descend(int i);
  // per-node exclusive device time (us) and peer bytes sent of one V-cycle, mean of `reps`
  void level_profile(int reps, std::vector<double>& us, std::vector<long long>& bytes);
  struct LevelProf {
    cudaEvent_t e[4]{};
    bool descended = false, recorded = false;
    long long bytes_in = 0, bytes_down = 0, bytes_up = 0, bytes_out = 0;
  };
  std::vector<LevelProf>* prof = nullptr;
  void smooth(int i, bool zero_x);
  void residual_restrict(int i, const Field& x);  // nodes[i+1].b = R (nodes[i].b - A x)
  void halo(int i, const Field& f);
  void apply(int i, const Field& x, const Field& y);
  void coarse_solve(int i);
  void estimate(int i, int mode);

  // collectives: per-box partials -> deterministic rank-ordered sums over dist (host)
  std::array<double, 2> collect2(int i, int nslots, const Field* a, const Field* b);
  void reduce_local(const Dist& D, int nslots, const Field* a, const Field* b, const Field* c, int nblk = 0);
  void device_allreduce_ranksums(int nslots);
  void zero_ranksums();
  void sync();  // drain the stream; throws if a cross-process barrier failed

  // compact (host or device) <-> field
  void upload(int i, const Field& f, const double* src, bool on_device);
  void download(int i, const Field& f, double* dst, bool on_device);

  cudaEvent_t caller_ev = nullptr;
  void order_after_caller();
  int solve(const double* b, double* x, bool on_device, int method, double rtol, double atol, int max_its,
            double* hist, int* reason, int* its, double* norm0, double* normf, double* t_ms, bool seeded,
            unsigned long long seed, bool x0_nonzero = true);

  // CG iteration as one CUDA graph (TMGX_GRAPHS=0 disables capture)
  bool use_graphs = true;
  bool tb_enabled = true;  // temporally blocked V(2,2) smoother (TMGX_TB=0 disables)
  bool tb3_enabled = true;  // temporally blocked V(3,3) smoother (TMGX_TB3=0 disables)
  int tb_min_extent = 0;    // blocked smoother only on levels at least this wide (TMGX_TB_MIN)
  bool fuse_dots = true;   // CG r.z, z.z from the finest blocked post-smooth (TMGX_FUSE_DOTS=0)
  int dots_nblk = 0;       // partials written by the last finest post-smooth (0: none)
  bool fuse_cg = true;     // p update fused into w = A p on single-box fine levels (TMGX_FUSE_CG=0)
  int fuse_rr2 = 1;        // performance build: separable fused residual + restriction on single-box levels.
                           // 1 (default): constant-coefficient rows only; 2: variable-coefficient rows too
                           // (2.7% faster on cfg3, but the re-associated sums move the 1e4-contrast 33^3
                           // solve to 1.04e-9 of the oracle, past the 1e-9 bar); 0: off (TMGX_FUSE_RR2)
  bool fuse_rr = false;    // fused residual + restriction on single-box levels (TMGX_FUSE_RR=1; measured
                           // slower than residual + restriction on B200)
  bool use_tb(int i) const;
  void tb_side(Node& nd, size_t q, const double* xin, double* xout, bool pre, bool dots = false);
  int cc_max_extent = 0;  // fused coarse V-cycle on single-box levels up to this size (TMGX_CC_MAX; off: measured
                          // no faster than per-phase launches)
  int cc_from = -1;        // first node of the fused coarse chain (set after setup)
  int coarse_chain_start() const;
  void coarse_cycle(int i0);
  ChebStep cheb_first_step(const Node& nd) const;
  cudaGraphExec_t iter_exec[2] = {nullptr, nullptr};  // one captured CG iteration per p parity
  long long iter_launches = 0;
  long long iter_bars = 0, graph_base = 0;
  void cg_dots(int op);
  void cg_iteration(int par);
  void run_iteration(int par);
  bool fused_cg() const;

 private:
  void build_nodes();
  void build_galerkin();
  void setup_coarse(Node& nd);
  double host_k(const Dist& D, long long gi, long long gj, long long gk) const;
};

}  // namespace tmgx
