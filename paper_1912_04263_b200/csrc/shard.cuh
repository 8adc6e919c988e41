// shard.cuh — the row-sharded solve: A cut into G
// contiguous nnz-balanced row blocks, each block a Workspace<T> holding A_g,
// its own transpose A_g^T (n x m_g), the replicated P and n-vectors, and the
// m_g-slices of every m-vector.  Per K-apply the only exchange is the sum of
// the A_g^T partial n-vectors; scalar decisions are taken from combined
// values, identical on every block, so the loop stays in lockstep without
// further communication.
//
// Exchanges per ADMM step (all through ShardComm):
//   rhs:   allreduce(2n)   [A^T (rho z - y), A^T (rho z~)]
//   PCG:   allreduce(n)    per iteration [A^T t]
//   check: allreduce(n) [A^T y] + allreduce_max(14 scalars)
//   rho:   allreduce_max(1) [|z|_inf]
//   infeasibility (rare): allreduce(3), allreduce(n), allreduce(1)
// Setup: allreduce_max(n) + allreduce_max(1) per Ruiz pass (maxima: the
// scaled problem stays bit-identical to the unsharded one) and a chain across
// blocks for diag(A^T A) (a sequential sum in the reference; chaining keeps
// it bit-exact), so the Jacobi preconditioner is bit-identical as well.
//
// The loop is host-driven: one control-block read per PCG iteration decides
// the next step on every block.
#pragma once

#include "comm.cuh"

namespace qpcg_b200 {

template <typename T>
class Sharded : public IEngine<T> {
 public:
  ShardComm comm;
  std::vector<std::unique_ptr<Workspace<T>>> sh;
  std::vector<uint32_t> cuts;      // [G + 1] global row cuts
  std::vector<uint32_t> rank_off;  // [R + 1] first row of every rank's blocks
  cudaStream_t s = nullptr;
  bool own_stream = true;
  int device = 0;
  uint32_t n = 0, m = 0;
  bool balanced = true;
  qpcg_options opt{};
  double setup_seconds = 0;
  uint64_t setup_launches = 0;
  bool have_counted_setup = false;
  T* full_m = nullptr;  // gather buffer [m]
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  Arena arena;  // the transient setup buffers of all blocks (one shared stream)
  ~Sharded() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    comm.free_p2p();  // a collective: every rank tears down together
    sh.clear();  // blocks free their buffers on the shared stream
    if (full_m) {
      AllocScope scope(s, &arena);
      dfree(full_m);
    }
    if (s) cudaStreamSynchronize(s);
    arena.return_all();
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (s && own_stream) cudaStreamDestroy(s);
  }

  Workspace<T>& w0() { return *sh[0]; }
  template <typename F>
  void each(F&& f) {
    for (auto& w : sh) f(*w);
  }
  template <typename U, typename F>
  std::vector<U*> bufs(F&& f) {
    std::vector<U*> v;
    for (auto& w : sh) v.push_back(f(*w));
    return v;
  }
  void allreduce_part(size_t count) {
    comm.allreduce(bufs<T>([](Workspace<T>& w) { return w.D.part; }), count, false);
  }
  void allreduce_scal(size_t count, bool max) {
    comm.allreduce(bufs<T>([](Workspace<T>& w) { return w.D.shsc; }), count, max);
  }
  // min of a per-block host key over every block of every rank
  unsigned long long agree_min(const std::vector<unsigned long long>& keys) {
    unsigned long long k = ~0ull;
    for (auto v : keys) k = std::min(k, v);
    if (comm.multi()) {
      unsigned long long* d = w0().template alloc<unsigned long long>(1);
      CK(cudaMemcpyAsync(d, &k, 8, cudaMemcpyHostToDevice, s));
      comm.allreduce_min_u64(d);
      CK(cudaMemcpyAsync(&k, d, 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    }
    return k;
  }

  // ------------------------------------------------------------- setup
  void setup(const HostCsr<T>& Pu, const T* q, const HostCsr<T>& A, const T* l, const T* u,
             const qpcg_settings& st, const qpcg_options& op) override {
    const double w0s = now_s();
    const uint64_t l0 = g_launches;
    opt = op;
    Workspace<T>::validate_settings(st);
    if (op.on_iteration)
      throw InvalidArgument("on_iteration: not available on a row-sharded workspace");
    device = op.device;
    if (device < 0) CK(cudaGetDevice(&device));
    CK(cudaSetDevice(device));
    if (op.stream != nullptr) {
      s = static_cast<cudaStream_t>(op.stream);
      own_stream = false;
    } else {
      CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    }
    CK(cudaEventCreate(&ev0));
    CK(cudaEventCreate(&ev1));
    CK(cudaEventRecord(ev0, s));
    comm.s = s;
    comm.local = op.virtual_shards > 1 ? op.virtual_shards : 1;
    if (comm.local > kMaxLocalShards) throw InvalidArgument("options: at most 16 virtual shards");
    const bool peer = op.transport == QPCG_TRANSPORT_PEER;
    if (op.nccl_id != nullptr || peer) {
      if (op.nccl_ranks < 1 || op.nccl_rank < 0 || op.nccl_rank >= op.nccl_ranks)
        throw InvalidArgument("options: bad rank / ranks");
      if (op.nccl_ranks > kMaxLocalShards) throw InvalidArgument("options: at most 16 ranks");
    }
    if (op.nccl_id != nullptr) comm.init_nccl(op.nccl_id, op.nccl_rank, op.nccl_ranks);
    n = Pu.rows;
    m = A.rows;
    if (peer) comm.init_p2p(op.nccl_rank, op.nccl_ranks, op.rendezvous_dir, n, m);
    const uint32_t L = comm.local, R = comm.nranks, G = L * R;
    // ---- nnz-balanced cuts from the (host copy of) row_ptr
    std::vector<uint32_t> hrp;
    const uint32_t* rp = A.row_ptr;
    if (op.input_memory != QPCG_MEM_HOST) {
      hrp.resize(size_t(m) + 1);
      CK(cudaMemcpyAsync(hrp.data(), A.row_ptr, 4 * (size_t(m) + 1), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      rp = hrp.data();
    }
    cuts.assign(G + 1, 0);
    balanced = shard_cuts(rp, m, A.nnz, G, cuts.data());
    rank_off.assign(R + 1, 0);
    for (uint32_t r = 0; r <= R; ++r) rank_off[r] = cuts[r * L];
    // ---- per-block upload and validation
    std::vector<unsigned long long> kp, ka, kv;
    for (uint32_t li = 0; li < L; ++li) {
      const int g = comm.global_index(li);
      sh.emplace_back(new Workspace<T>());
      Workspace<T>& w = *sh.back();
      w.D.split = 1;
      w.D.sh_index = g;
      w.D.sh_count = G;
      w.begin(st, op, s);
      AllocScope scope(s, &arena);
      if (balanced)
        w.load(Pu, q, A, l, u, cuts[g], cuts[g + 1], true);
      else if (g == 0)  // invalid row_ptr: block 0 sees A exactly as given
        w.load(Pu, q, A, l, u, 0, m, false);
      else
        w.load(Pu, q, A, l, u, m, m, true);
      const typename Workspace<T>::ValKeys v = w.validate_keys();
      // P's row_ptr ends are identical on every block; A's are block-local
      // (and only block 0 can see a bad one): fold both into the stage keys
      // (0 = "row_ptr must start at 0 and end at nnz", ahead of any key)
      kp.push_back((v.ends[0] != 0 || v.ends[1] != w.pu_nnz) ? 0ull : v.k[0]);
      ka.push_back((v.ends[2] != 0 || v.ends[3] != w.D.A.nnz) ? 0ull : v.k[1]);
      kv.push_back(v.k[2]);
    }
    {
      typename Workspace<T>::ValKeys v{};
      v.k[0] = agree_min(kp);
      v.k[1] = agree_min(ka);
      v.k[2] = agree_min(kv);
      if (v.k[0] == 0) throw InvalidArgument("csr: row_ptr must start at 0 and end at nnz");
      if ((v.k[0] >> 56) == kValPRowPtr) throw InvalidArgument(validation_message(v.k[0]));
      if (v.k[1] == 0) throw InvalidArgument("csr: row_ptr must start at 0 and end at nnz");
      // the rest of the reference order (problem.hpp:46-92) as raise_first
      Workspace<T>& w = w0();
      if ((v.k[1] >> 56) == kValARowPtr) throw InvalidArgument(validation_message(v.k[1]));
      if (!w.p_square) throw InvalidArgument("problem: P must be square");
      if (n == 0) throw InvalidArgument("problem: at least one variable required");
      if ((v.k[0] >> 56) == kValPBelow) throw InvalidArgument(validation_message(v.k[0]));
      if (!w.a_cols_ok) throw InvalidArgument("problem: A column count must equal n");
      if (v.k[2] != ~0ull) throw InvalidArgument(validation_message(v.k[2]));
    }
    AllocScope scope(s, &arena);
    each([](Workspace<T>& w) { w.build_structures(); });
    // ---- Ruiz with the two maxima combined across blocks
    uint32_t passes = 0;
    T deviation = T(0);
    if (st.scaling_enabled) {
      each([](Workspace<T>& w) { w.ruiz_prepare(); });
      deviation = T(1);
      while (passes < st.equil_max_passes && deviation > T(st.eps_equil)) {
        ++passes;
        each([](Workspace<T>& w) { w.ruiz_norms(); });
        comm.allreduce(bufs<T>([](Workspace<T>& w) { return w.rz_atn; }), n, true);
        each([](Workspace<T>& w) { w.ruiz_delta(); });
        comm.allreduce(bufs<T>([](Workspace<T>& w) { return w.ruiz_scal + 4; }), 1, true);
        each([](Workspace<T>& w) { w.ruiz_scale(); });
        deviation = w0().read_scalar(w0().ruiz_scal + 4);
      }
    }
    each([&](Workspace<T>& w) { w.finish_scaling(passes, deviation); });
    // ---- diag(A^T A): one sequential chain through the blocks in row order
    T* acc = w0().D.diag_ata;
    comm.chain(acc, n, [&] {
      for (uint32_t li = 0; li < L; ++li) {
        const bool first = comm.rank == 0 && li == 0;
        diag_ata_kernel<T><<<grid_for(uint64_t(n) * 32), kThreads, 0, s>>>(sh[li]->D.AT, acc,
                                                                            first ? nullptr : acc);
        CK_LAUNCH();
      }
    });
    for (uint32_t li = 1; li < L; ++li)
      CK(cudaMemcpyAsync(sh[li]->D.diag_ata, acc, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
    each([](Workspace<T>& w) { w.finish_setup(); });
    CK(dmalloc(&full_m, sizeof(T) * (size_t(m) + 1)));
    CK(cudaEventRecord(ev1, s));
    CK(cudaEventSynchronize(ev1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev0, ev1));
    setup_seconds = ms * 1e-3;
    each([&](Workspace<T>& w) {
      w.setup_seconds = setup_seconds;
      w.setup_wall = now_s() - w0s;
    });
    setup_launches = g_launches - l0;
  }

  // ------------------------------------------------------ loop pieces
  // A^T pass of block w into the partial buffers, combined over all blocks:
  // with the peer transport the epilogue stores into every rank's slot (the
  // fused compute + collective), else EpiPart + the comm's allreduce.
  template <int NCOL, class Gather>
  void at_pass_combined(Workspace<T>& w, int li, const Gather& g, uint32_t gate) {
    if (comm.p2p)
      launch_spmv<T, NCOL, SumOp>(w.D.AT, w.D.pAT, g,
                                  EpiPeer<T, NCOL>{comm.p2p_slot(li), comm.p2p->R, w.D.ctl, gate,
                                                   comm.p2p->vec_set(), comm.dev_epoch(), 0},
                                  w.s);
    else
      launch_spmv<T, NCOL, SumOp>(w.D.AT, w.D.pAT, g, EpiPart<T, NCOL>{w.D.part, w.D.ctl, gate}, w.s);
  }
  void combine_parts(size_t count) {
    if (comm.p2p)
      comm.p2p_reduce(bufs<T>([](Workspace<T>& w) { return w.D.part; }), count, false);
    else
      allreduce_part(count);
  }

  void enq_rhs(Handles H = {}) {
    int li = 0;
    each([&](Workspace<T>& w) {
      k_pack_rhs<T><<<grid_for(w.D.m), kThreads, 0, w.s>>>(w.D);
      CK_LAUNCH();
      at_pass_combined<2>(w, li++, GatherRhs<T>{w.D.g2m}, 0);
    });
    combine_parts(2 * size_t(n));
    each([&](Workspace<T>& w) {
      k_rhs_finish<T><<<grid_for(w.D.n), kThreads, 0, w.s>>>(w.D);
      CK_LAUNCH();
      w.enq_pcg_init(H);
    });
  }
  void enq_pcg_iter(Handles H = {}) {
    int li = 0;
    each([&](Workspace<T>& w) {
      launch_spmv<T, 1, SumOp>(w.D.A, w.D.pA, GatherVec<T>{w.D.p}, EpiAp<T>{w.D.t, w.D.ap, w.D.ctl}, w.s);
      at_pass_combined<1>(w, li++, GatherVec<T>{w.D.t}, 1);
    });
    combine_parts(n);
    each([&](Workspace<T>& w) {
      k_pcg_dot<T><<<red_grid<T>(w.D.n), kThreads, 0, w.s>>>(w.D);
      CK_LAUNCH();
      k_pcg_update<T><<<red_grid<T>(w.D.n), kThreads, 0, w.s>>>(w.D, H);
      CK_LAUNCH();
      k_pcg_pupdate<T><<<grid_for(w.D.n), kThreads, 0, w.s>>>(w.D);
      CK_LAUNCH();
    });
  }
  void enq_check(int mode, Handles H = {}) {
    int li = 0;
    each([&](Workspace<T>& w) { at_pass_combined<1>(w, li++, GatherVec<T>{w.D.y}, 0); });
    combine_parts(n);
    each([&](Workspace<T>& w) {
      k_dual_finish<T><<<grid_for(w.D.n), kThreads, 0, w.s>>>(w.D);
      CK_LAUNCH();
      k_residuals<T><<<red_grid<T>(std::max(w.D.n, w.D.m)), kThreads, 0, w.s>>>(w.D, mode, Handles{});
      CK_LAUNCH();
    });
    allreduce_scal(14, true);
    each([&](Workspace<T>& w) {
      k_residuals_decide<T><<<1, 32, 0, w.s>>>(w.D, mode, H);
      CK_LAUNCH();
    });
  }
  void enq_residuals_fresh(int mode) {
    each([](Workspace<T>& w) {
      launch_spmv<T, 1, SumOp>(w.D.A, w.D.pA, GatherVec<T>{w.D.x}, EpiStore<T>{w.D.ax}, w.s);
    });
    enq_check(mode);
  }
  void enq_infeas() {
    each([](Workspace<T>& w) {
      k_infeas_vec<T><<<red_grid<T>(std::max(w.D.n, w.D.m)), kThreads, 0, w.s>>>(w.D);
      CK_LAUNCH();
    });
    allreduce_scal(3, false);
    each([](Workspace<T>& w) {
      Dev<T>& D = w.D;
      k_infeas_vec_decide<T><<<1, 32, 0, w.s>>>(D);
      CK_LAUNCH();
      launch_spmv<T, 1, SumOp>(D.ATo, D.pATo, GatherCertY<T>{D.e, D.dy, D.ctl, T(0), T(0)},
                               EpiPart<T, 1>{D.part, D.ctl, 2}, w.s);
    });
    allreduce_part(n);
    each([](Workspace<T>& w) {
      Dev<T>& D = w.D;
      k_atv_norm<T><<<red_grid<T>(D.n), kThreads, 0, w.s>>>(D);
      CK_LAUNCH();
      launch_spmv<T, 1, SumOp>(D.Po, D.pPo, GatherCertX<T>{D.d, D.dx, D.ctl, T(0)},
                               EpiNormMax<T>{&D.ctl->pv_inf_bits, &D.ctl->need_dinf}, w.s);
      k_infeas_mid<T><<<1, 1, 0, w.s>>>(D);
      CK_LAUNCH();
      launch_spmv<T, 1, SumOp>(
          D.Ao, D.pAo, GatherCertX<T>{D.d, D.dx, D.ctl, T(0)},
          EpiDualRows<T>{D.l_o, D.u_o, &D.ctl->dinf_bad, &D.ctl->need_dinf, T(0), D.ctl}, w.s);
      k_flag_to_scal<T><<<1, 1, 0, w.s>>>(D);
      CK_LAUNCH();
    });
    allreduce_scal(1, false);
    each([](Workspace<T>& w) {
      k_infeas<T><<<1, 1, 0, w.s>>>(w.D);
      CK_LAUNCH();
    });
  }
  void enq_rho() {
    each([](Workspace<T>& w) {
      w.enq_rho_flag(Handles{});  // (no IF node: the rho kernels gate themselves)
      k_rho<T><<<red_grid<T>(w.D.m), kThreads, 0, w.s>>>(w.D);
      CK_LAUNCH();
    });
    allreduce_scal(1, true);
    each([](Workspace<T>& w) {
      k_rho_decide<T><<<1, 32, 0, w.s>>>(w.D);
      CK_LAUNCH();
      k_precond<T><<<grid_for(w.D.n), kThreads, 0, w.s>>>(w.D, 0);
      CK_LAUNCH();
    });
  }

  // ------------------------------------------------- device-driven loop
  // The same sequence as the host loop below as one CUDA graph with
  // conditional WHILE / IF nodes: the decisions come from the (identical)
  // control blocks of the row blocks, the collectives are kernels (local
  // combine, peer stores, device barriers), so nothing returns to the host
  // until the solve ends.  Not with the NCCL transport.
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  bool graph_ok() const { return opt.mode == QPCG_MODE_GRAPH && (comm.p2p || !comm.comm); }
  cudaGraph_t add_cond(cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type) {
    cudaStreamCaptureStatus cs;
    cudaGraph_t g;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &nd));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = type;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, deps, nd, &cp));
    CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    return cp.conditional.phGraph_out[0];
  }
  void build_graph() {
    CK(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle h_admm, h_pcg, h_chk, h_inf;
    CK(cudaGraphConditionalHandleCreate(&h_admm, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h_admm;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t n_admm;
    CK(cudaGraphAddNode(&n_admm, graph, nullptr, 0, &cp));
    cudaGraph_t b_admm = cp.conditional.phGraph_out[0];
    CK(cudaGraphConditionalHandleCreate(&h_pcg, b_admm, 0, cudaGraphCondAssignDefault));
    CK(cudaGraphConditionalHandleCreate(&h_chk, b_admm, 0, cudaGraphCondAssignDefault));
    Handles H;
    H.admm = (unsigned long long)h_admm;
    H.pcg = (unsigned long long)h_pcg;
    H.chk = (unsigned long long)h_chk;
    cudaGraph_t b_pcg, b_chk, b_inf, g_out;
    // kernels per execution of each body, counted as they are captured
    const uint64_t b0 = g_launches;
    uint64_t c0 = g_launches;
    CK(cudaStreamBeginCaptureToGraph(s, b_admm, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    enq_rhs(H);
    b_pcg = add_cond(h_pcg, cudaGraphCondTypeWhile);
    each([&](Workspace<T>& w) { w.enq_post_pcg(H); });
    b_chk = add_cond(h_chk, cudaGraphCondTypeIf);
    enq_rho();
    each([&](Workspace<T>& w) { w.enq_admm_cond(H); });
    CK(cudaStreamEndCapture(s, &g_out));
    body_kernels[0] = g_launches - c0;
    c0 = g_launches;
    CK(cudaStreamBeginCaptureToGraph(s, b_pcg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    enq_pcg_iter(H);
    CK(cudaStreamEndCapture(s, &g_out));
    body_kernels[1] = g_launches - c0;
    CK(cudaGraphConditionalHandleCreate(&h_inf, b_chk, 0, cudaGraphCondAssignDefault));
    H.inf = (unsigned long long)h_inf;
    c0 = g_launches;
    CK(cudaStreamBeginCaptureToGraph(s, b_chk, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    enq_check(0, H);
    b_inf = add_cond(h_inf, cudaGraphCondTypeIf);
    CK(cudaStreamEndCapture(s, &g_out));
    body_kernels[2] = g_launches - c0;
    c0 = g_launches;
    CK(cudaStreamBeginCaptureToGraph(s, b_inf, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    enq_infeas();
    CK(cudaStreamEndCapture(s, &g_out));
    body_kernels[3] = g_launches - c0;
    graph_build = g_launches - b0;  // captured, not launched
    CK(cudaGraphInstantiate(&exec, graph, 0));
  }
  uint64_t body_kernels[4] = {};  // per execution: ADMM step, PCG iteration, check, infeas
  uint64_t graph_build = 0;

  // ------------------------------------------------------------ solve
  void solve(qpcg_info* info, T* x, T* z, T* y, T* cert) override {
    CK(cudaSetDevice(device));
    AllocScope scope(s, &arena);
    const double w0s = now_s();
    CK(cudaEventRecord(ev0, s));
    each([](Workspace<T>& w) { w.reset_solve_state(); });
    const uint64_t l0 = g_launches;
    Workspace<T>& W = w0();
    enq_residuals_fresh(1);  // solver.hpp:436-441
    uint64_t graph_built_now = 0;
    if (graph_ok()) {
      if (!exec) {
        build_graph();
        graph_built_now = graph_build;
      }
      CK(cudaGraphLaunch(exec, s));
    }
    for (; !graph_ok();) {
      W.pull_ctl();
      if (W.hc.done || W.hc.error || W.hc.iter >= W.hc.max_iter) break;
      enq_rhs();
      W.pull_ctl();
      while (W.hc.pcg_active && !W.hc.error) {
        enq_pcg_iter();
        W.pull_ctl();
      }
      each([](Workspace<T>& w) { w.enq_post_pcg(Handles{}); });
      W.pull_ctl();
      if (W.hc.is_check && !W.hc.error) {
        enq_check(0);
        W.pull_ctl();
        if (W.hc.inf_branch) enq_infeas();
      }
      enq_rho();
    }
    W.pull_ctl();
    W.raise_device_error();
    if (!W.hc.residuals_current) enq_residuals_fresh(2);
    each([](Workspace<T>& w) {
      Dev<T>& D = w.D;
      k_unscale<T><<<grid_for(std::max(D.n, D.m)), kThreads, 0, w.s>>>(D);
      CK_LAUNCH();
    });
    W.pull_ctl();
    const bool infeasible = W.hc.status == 1 || W.hc.status == 2;
    if (!infeasible)  // P is replicated: block 0 alone forms the objective
      launch_spmv<T, 1, SumOp>(W.D.Po, W.D.pPo, GatherVec<T>{W.D.xo}, EpiStore<T>{W.D.pxo}, s);
    k_objective<T><<<red_grid<T>(n), kThreads, 0, s>>>(W.D);
    CK_LAUNCH();
    CK(cudaEventRecord(ev1, s));
    W.pull_ctl();
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev0, ev1));
    // m-side outputs: every block's slice at its global rows, then across ranks
    const double td0 = now_s();
    gather_m([](Workspace<T>& w) { return w.D.zo; }, z);
    gather_m([](Workspace<T>& w) { return w.D.yo; }, y);
    W.download(x, W.D.xo, sizeof(T) * n);
    if (W.hc.status == 1)
      gather_m([](Workspace<T>& w) { return w.D.cert; }, cert);
    else if (W.hc.status == 2)
      W.download(cert, W.D.cert, sizeof(T) * n);
    CK(cudaStreamSynchronize(s));
    const double d2h = now_s() - td0;
    if (info) {
      W.fill_info(info, ms * 1e-3, d2h, n, m);
      info->setup_seconds = setup_seconds;
      info->runtime_seconds = now_s() - w0s;
      uint64_t h2d = 0;
      double h2ds = 0;
      each([&](Workspace<T>& w) {
        h2d += w.h2d_bytes;
        h2ds += w.h2d_seconds;
      });
      info->h2d_bytes = h2d;
      info->h2d_seconds = h2ds;
      uint64_t launches = g_launches - l0 - graph_built_now;
      if (graph_ok())  // kernels executed inside the graph
        launches += W.hc.iter * body_kernels[0] + W.hc.pcg_total * body_kernels[1] +
                    uint64_t(W.hc.n_checks) * body_kernels[2] + uint64_t(W.hc.n_inf) * body_kernels[3];
      info->kernel_launches = launches + (have_counted_setup ? 0 : setup_launches);
    }
    have_counted_setup = true;
  }

  // download (host or device destination) an m-vector assembled from the blocks
  template <typename F>
  void gather_m(F&& src, T* dst) {
    if (dst == nullptr || m == 0) return;
    each([&](Workspace<T>& w) {
      if (w.D.m)
        CK(cudaMemcpyAsync(full_m + w.row0, src(w), sizeof(T) * w.D.m, cudaMemcpyDeviceToDevice, s));
    });
    comm.allgather_blocks(full_m, rank_off);
    w0().download(dst, full_m, sizeof(T) * m);
  }

  // ------------------------- diagnostics / debug: the first row block
  uint32_t pcg_calls(qpcg_pcg_call* out, uint32_t cap) override { return w0().pcg_calls(out, cap); }
  uint32_t rho_updates(qpcg_rho_update* out, uint32_t cap) override {
    return w0().rho_updates(out, cap);
  }
  uint32_t check_iterations(uint32_t* out, uint32_t cap) override {
    return w0().check_iterations(out, cap);
  }
  void dims(uint64_t* d) override {
    w0().dims(d);
    d[1] = m;  // global m; nnz(A) of every block summed
    uint64_t nnz = 0;
    each([&](Workspace<T>& w) { nnz += w.D.A.nnz; });
    d[3] = nnz;
  }
  void debug_scaled(T*, uint32_t*, uint32_t*, T*, T*, T*, uint32_t*, uint32_t*, T*, T*, T*, T*,
                    double*) override {
    throw InvalidArgument("debug_scaled: not available on a row-sharded workspace");
  }
  void debug_operator(const T*, T*, T*) override {
    throw InvalidArgument("debug_operator: not available on a row-sharded workspace");
  }
  void bench_kernels(uint32_t reps, double* out) override { w0().bench_kernels(reps, out); }

  // --------------------------------------------------- OSQP-style updates
  void warm_start(const T* x, const T* z, const T* y) override {
    CK(cudaSetDevice(device));
    AllocScope scope(s, &arena);
    std::vector<unsigned long long> keys;
    each([&](Workspace<T>& w) { keys.push_back(w.warm_stage(x, z + w.row0, y + w.row0)); });
    if (agree_min(keys) != ~0ull) throw InvalidArgument("solve: warm start must be finite");
    each([](Workspace<T>& w) { w.warm_apply(); });
  }
  void update_rho(T rho) override {
    each([&](Workspace<T>& w) { w.update_rho(rho); });
  }
  void update_vectors(const T* q, const T* l, const T* u) override {
    CK(cudaSetDevice(device));
    AllocScope scope(s, &arena);
    std::vector<unsigned long long> keys;
    each([&](Workspace<T>& w) {
      keys.push_back(w.vectors_stage(q, l ? l + w.row0 : nullptr, u ? u + w.row0 : nullptr));
    });
    const unsigned long long k = agree_min(keys);
    if (k != ~0ull) throw InvalidArgument(validation_message(k));
    each([](Workspace<T>& w) { w.vectors_apply(); });
  }
};

}  // namespace qpcg_b200
