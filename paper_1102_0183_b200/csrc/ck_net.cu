// ck_net.cu — the network seam: device-resident nets, the persistent team
// kernel that runs whole online epochs, batched evaluation, and the C ABI
// (ck_net_* / ck_committee_*) declared in include/ckb200.h.
//
// Replaces, behind the reference's API, NetworkState (network.py:81-304)
// and the per-image loops of training.train_epoch / evaluate
// (training.py:126-156).  One launch processes a whole sequence of images:
// for each image the team runs the phases of PROG_TRAIN (forward, output
// delta, backward with in-place updates) separated by team barriers.
#include <cooperative_groups.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "ck_host.h"
#include "ck_kernels.cuh"
#ifndef CK_NO_SPECS
#include "ck_specs.inc"   // generated: the specialised nets (tools/gen_specs.py)
#else
#define CK_SPEC_LIST(X)   // stage-1 build (the generator's own library)
#endif

namespace ck {
// one per spec, defined in its generated translation unit ck_spec_<name>.cu
#define CK_SPEC_DECL(S) const void* spec_kernel_##S(); const void* spec_eval_kernel_##S();
CK_SPEC_LIST(CK_SPEC_DECL)
#undef CK_SPEC_DECL
}  // namespace ck

// ===========================================================================
// host runtime

using namespace ck;

struct ck_net {
  int device = 0;
  NetGeo h;                       // geometry + programs (host image)
  NetGeo* d_desc = nullptr;       // device copy (read by the generic kernels)
  NetPtr ptr;                     // device memory of the net
  int spec = -1;                  // index in spec_table() (-1: generic kernel only)
  int use_spec = 1;               // ck_net_set_specialized
  float* d_params = nullptr;
  float* d_grads = nullptr;
  float* d_act = nullptr;
  int* d_tables = nullptr;
  double* d_filters = nullptr;
  unsigned* d_bar = nullptr;
  double* d_targets = nullptr;    // single-step staging
  double* d_loss = nullptr;       // per-launch loss total (1 double)
  float* d_eval = nullptr;        // eval scratch arenas
  float* d_pre = nullptr;         // training: precomputed image-processing layers
  int64_t pre_cap = 0;            // floats
  int eval_ctas = 0;
  int64_t n_params = 0;
  int team_kind = CK_TEAM_AUTO;   // resolved per launch (resolve_team)
  int team_ctas = 0;
  int threads = 512;
  cudaStream_t stream = nullptr;  // private stream for the synchronous calls
  std::vector<int64_t> grad_count;  // per layer (params it owns)
};

namespace {

int64_t align32(int64_t v) { return (v + 31) & ~int64_t(31); }

struct ProgramBuilder {
  Program& p;
  explicit ProgramBuilder(Program& prog) : p(prog) {
    memset(&p, 0, sizeof(Program));
  }
  int n_ops = 0;
  std::vector<Op> cur;
  bool ok = true;
  void add(int kind, int layer, int flags = 0) {
    Op o;
    o.kind = (int16_t)kind;
    o.layer = (int16_t)layer;
    o.flags = (int16_t)flags;
    o.pad = 0;
    cur.push_back(o);
  }
  void phase() {
    if (cur.empty()) return;
    if (p.n_phases >= kMaxPhases || n_ops + (int)cur.size() > kMaxOps) {
      ok = false;
      cur.clear();
      return;
    }
    p.begin[p.n_phases] = n_ops;
    for (const Op& o : cur) p.ops[n_ops++] = o;
    p.n_phases++;
    p.begin[p.n_phases] = n_ops;
    cur.clear();
  }
};

// `skip_out`: the output layer's forward is folded into OP_FC_OUT.
void build_forward(ProgramBuilder& b, const NetGeo& N, bool load, bool zero,
                   bool skip_out = false, bool pooled_only = false) {
  const int last = skip_out ? N.n_layers - 1 : N.n_layers;
  // The first layer can read the image itself (stage_input) when it is a
  // conv+pool or the contrast layer and the image fits in shared memory; the
  // input copy for later phases is then published in that same phase.
  const bool fold = load && N.in_cells <= 8192 && N.n_layers > 2 &&
                    ((N.L[1].kind == L_CONV && 2 < last && N.L[2].kind == L_POOL) ||
                     N.L[1].kind == L_IMGPROC);
  if (load && !fold) {
    b.add(OP_LOAD_INPUT, 0);
    b.phase();
  }
  if (fold) b.add(OP_LOAD_INPUT, 0);
  for (int k = 1; k < last; ++k) {
    const LayerDev& L = N.L[k];
    const bool scatter_target = zero && k + 1 < N.n_layers &&
                                N.L[k + 1].kind == L_POOL && L.has_delta;
    if (L.kind == L_CONV && k + 1 < last && N.L[k + 1].kind == L_POOL) {
      // conv + the max-pool above it in one phase
      b.add(OP_CONV_POOL, k, (scatter_target ? F_ZERO_SELF : 0) | (pooled_only ? F_POOLED_ONLY : 0));
      const bool pool_target = zero && k + 2 < N.n_layers && N.L[k + 2].kind == L_POOL;
      if (pool_target) b.add(OP_ZERO_DELTA, k + 1);
      b.phase();
      ++k;
      continue;
    }
    switch (L.kind) {
      case L_IMGPROC: b.add(OP_IMGPROC, k); break;
      case L_CONV: b.add(OP_CONV_FWD, k, scatter_target ? F_ZERO_SELF : 0); break;
      case L_POOL:
        b.add(OP_POOL_FWD, k);
        if (scatter_target) b.add(OP_ZERO_DELTA, k);
        break;
      case L_FC: b.add(OP_FC_FWD, k); break;
      default: break;
    }
    b.phase();
  }
}

// Backward walk of network.py:205-262 as phases.  With `update`, each
// learnable layer is updated as soon as nothing later reads its old weights:
// FC rows in place, a conv whose pull is done in the following phase.
void build_backward(ProgramBuilder& b, const NetGeo& N, bool update) {
  std::vector<int> pending;
  int k = N.n_layers - 1;
  bool done = false;
  while (!done && k >= 1 && N.L[k].kind == L_FC) {
    // every CTA reads the whole output layer in OP_FC_OUT, so its update
    // waits for the next phase
    const bool out = k == N.n_layers - 1;
    if (out && k >= 2 && N.L[k - 1].kind == L_FC && N.L[k - 1].cells <= kFuseHiddenMax &&
        N.L[k - 2].kind != L_INPUT) {
      // output layer + the hidden FC below it in one phase (F_FUSE_BELOW)
      b.add(OP_FC_OUT, k, F_FUSE_BELOW | (update ? F_UPDATE : 0));
      for (int u : pending) b.add(OP_UPDATE, u);
      pending.clear();
      if (update) pending.push_back(k);
      b.phase();
      k -= 2;
      if (!N.L[k].has_delta) done = true;
      continue;
    }
    b.add(out ? OP_FC_OUT : OP_FC_BWD, k, (update && !out) ? F_UPDATE : 0);
    for (int u : pending) b.add(OP_UPDATE, u);
    pending.clear();
    if (update && out) pending.push_back(k);
    b.phase();
    --k;
    if (!N.L[k].has_delta) done = true;
  }
  while (!done && k >= 1) {
    const LayerDev& L = N.L[k];
    if (L.kind == L_CONV) {
      const bool pull = N.L[k - 1].has_delta;
      int flags = pull ? F_PULL : 0;
      if (update && !pull) flags |= F_UPDATE;
      b.add(OP_CONV_BWD, k, flags);
      for (int u : pending) b.add(OP_UPDATE, u);
      pending.clear();
      b.phase();
      if (update && pull) pending.push_back(k);
      if (!pull) break;
    } else if (L.kind == L_POOL) {
      if (!N.L[k - 1].has_delta) break;
    } else {
      break;
    }
    --k;
  }
  for (int u : pending) b.add(OP_UPDATE, u);
  b.phase();
}

void build_programs(NetGeo& N, bool* ok) {
  {
    ProgramBuilder b(N.prog[PROG_TRAIN]);
    build_forward(b, N, true, true, true);
    build_backward(b, N, true);
    *ok = *ok && b.ok;
  }
  {
    ProgramBuilder b(N.prog[PROG_FORWARD]);
    build_forward(b, N, false, true);
    *ok = *ok && b.ok;
  }
  {
    ProgramBuilder b(N.prog[PROG_BACKWARD]);
    build_backward(b, N, false);
    *ok = *ok && b.ok;
  }
  {
    ProgramBuilder b(N.prog[PROG_APPLY]);
    for (int k = 1; k < N.n_layers; ++k)
      if (N.L[k].n_par > 0) b.add(OP_UPDATE, k);
    b.phase();
    *ok = *ok && b.ok;
  }
  {
    ProgramBuilder b(N.prog[PROG_EVAL]);
    build_forward(b, N, true, false, false, true);
    *ok = *ok && b.ok;
  }
}

size_t team_smem_bytes() { return kDescBytes + kScratchBytes + kTeamStageFloats * sizeof(float); }
size_t eval_smem_bytes(int floats = kEvalBigFloats) { return kDescBytes + floats * sizeof(float); }

// Wide nets (a source layer beyond half the 2-CTA budget) evaluate with one
// CTA per SM and the whole shared memory; the rest with two.
int eval_floats_for(const NetGeo& N) {
  int widest = 0;
  for (int k = 1; k < N.n_layers; ++k) widest = std::max(widest, N.L[k].src_cells);
  return widest > kEvalStageFloats / 2 ? kEvalBigFloats : kEvalStageFloats;
}

int configure_kernels() {
  static bool done = false;
  if (done) return CK_OK;
  const int smem = (int)team_smem_bytes();
  CK_CUDA_TRY(cudaFuncSetAttribute(net_team_kernel<ClusterTeam>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK_CUDA_TRY(cudaFuncSetAttribute(net_team_kernel<ClusterTeam>,
                                   cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK_CUDA_TRY(cudaFuncSetAttribute(net_team_kernel<GridTeam>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK_CUDA_TRY(cudaFuncSetAttribute(net_eval_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)eval_smem_bytes()));
  done = true;
  return CK_OK;
}

struct SpecEntry {
  const char* name;
  NetGeo geo;
  const void* kernel;        // net_spec_kernel<Spec, GridTeam>
  const void* eval_kernel;   // net_eval_spec_kernel<Spec>
};

#define CK_SPEC_ENTRY(S) {#S, S::geo(), spec_kernel_##S(), spec_eval_kernel_##S()},
const SpecEntry* spec_table(int* n) {
  static const SpecEntry table[] = {
      CK_SPEC_LIST(CK_SPEC_ENTRY){nullptr, NetGeo{}, nullptr, nullptr}};
  *n = (int)(sizeof(table) / sizeof(table[0])) - 1;
  return table;
}
#undef CK_SPEC_ENTRY

int configure_spec_kernel(const void* kernel) {
  static std::vector<const void*> done;
  for (const void* k : done)
    if (k == kernel) return CK_OK;
  CK_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)team_smem_bytes()));
  done.push_back(kernel);
  return CK_OK;
}

// The team a launch of n_nets nets uses.  AUTO = a cooperative grid team
// spanning the whole GPU: one 512-thread CTA per SM, the SMs shared evenly
// between the nets of a committee (measured faster than 16-CTA clusters on
// every BASELINE configuration: more SMs for the wide phases, and a ~1.1 us
// arrival-counter barrier).
struct TeamShape {
  int kind, ctas, threads;
};

TeamShape resolve_team(const ck_net* net, int n_nets) {
  if (net->team_kind != CK_TEAM_AUTO) return {net->team_kind, net->team_ctas, net->threads};
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, net->device);
  return {CK_TEAM_GRID, std::max(1, sms / std::max(1, n_nets)), 512};
}

long long* g_sub = nullptr;   // ck_debug_subprof
int g_sub_rank = 0;

int launch_teams(ck_net* const* nets, int n_nets, Job job, cudaStream_t st) {
  job.sub = g_sub;
  job.sub_rank = g_sub_rank;
  int rc = configure_kernels();
  if (rc) return rc;
  const TeamShape t0 = resolve_team(nets[0], n_nets);
  NetRefs ptrs;
  memset(&ptrs, 0, sizeof(ptrs));
  for (int i = 0; i < n_nets; ++i) {
    const TeamShape ti = resolve_team(nets[i], n_nets);
    if (ti.kind != t0.kind || ti.ctas != t0.ctas || ti.threads != t0.threads)
      return set_error(CK_E_CONFIG, "all nets of one launch need the same team config");
    ptrs.geo[i] = nets[i]->d_desc;
    ptrs.ptr[i] = nets[i]->ptr;
  }
  job.n_nets = n_nets;
  const int ctas = t0.ctas;
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(ctas * n_nets);
  cfg.blockDim = dim3(t0.threads);
  cfg.dynamicSmemBytes = team_smem_bytes();
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  // the specialised kernel when every net of the launch has the same spec
  const void* spec_kernel = nullptr;
  if (t0.kind == CK_TEAM_GRID && job.prog == PROG_TRAIN && nets[0]->spec >= 0) {
    bool same = true;
    for (int i = 0; i < n_nets; ++i)
      same = same && nets[i]->spec == nets[0]->spec && nets[i]->use_spec;
    // an explicit team must match the specialised kernel's block size
    same = same && (nets[0]->team_kind == CK_TEAM_AUTO || t0.threads == CK_SPEC_THREADS);
    if (same) {
      int n_spec = 0;
      spec_kernel = spec_table(&n_spec)[nets[0]->spec].kernel;
      rc = configure_spec_kernel(spec_kernel);
      if (rc) return rc;
    }
  }
  if (spec_kernel && nets[0]->team_kind == CK_TEAM_AUTO) cfg.blockDim = dim3(CK_SPEC_THREADS);
  if (t0.kind == CK_TEAM_GRID) {
    for (int i = 0; i < n_nets; ++i) {   // arrival counters start at 0 every launch
      e = cudaMemsetAsync(nets[i]->d_bar, 0, 2 * sizeof(unsigned), st);
      if (e != cudaSuccess) return cuda_status(e, "reset grid barrier");
    }
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    if (spec_kernel) {
      void* args[] = {&ptrs, &job, (void*)&ctas};
      e = cudaLaunchKernelExC(&cfg, spec_kernel, args);
    } else {
      e = cudaLaunchKernelEx(&cfg, net_team_kernel<GridTeam>, ptrs, job, ctas);
    }
  } else {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ctas;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    e = cudaLaunchKernelEx(&cfg, net_team_kernel<ClusterTeam>, ptrs, job, ctas);
  }
  count_launch();
  if (e != cudaSuccess) return cuda_status(e, "net_team_kernel launch");
  return CK_OK;
}

Job empty_job(int prog) {
  Job j;
  memset(&j, 0, sizeof(j));
  j.prog = prog;
  j.n = 1;
  return j;
}

// The per-sample / host-buffer API runs on the net's private stream; work a
// caller enqueued on ITS streams (ck_net_train_epoch, ck_net_eval, ... with a
// user stream) may still be reading or writing this net.  Every synchronous
// entry therefore waits for the whole device first (no ordering
// existed between the two), and ends with its own stream drained.
int quiesce(ck_net* net) {
  CK_CUDA_TRY(cudaSetDevice(net->device));
  CK_CUDA_TRY(cudaDeviceSynchronize());
  return CK_OK;
}

int run_single(ck_net* net, Job job) {
  CK_CUDA_TRY(cudaSetDevice(net->device));
  job.loss_total = net->d_loss;
  job.full = 1;   // per-sample API: every buffer is readable afterwards
  int rc = launch_teams(&net, 1, job, net->stream);
  if (rc) return rc;
  CK_CUDA_TRY(cudaStreamSynchronize(net->stream));
  return CK_OK;
}

// Row pitch for a conv's source layer staged whole in shared memory
// (conv_pool_fwd): the lanes of a warp take consecutive cells of pool blocks
// (one cell each, reference-order chain) and at every step all read the same
// tap of their own window; the pitch decides which banks those addresses hit.
// Pick the smallest pitch in [w, w + 32) minimising the shared-memory
// wavefronts of one such load, summed over the warps of a 148-CTA team.
// Performance only: every pitch gives the same bits.
static int choose_src_pitch(const LayerDev& L, const LayerDev& S, const LayerDev& P) {
  const int blk = P.px * P.py, phw = P.h * P.w, team = 148;
  int best_pitch = S.w;
  long best = -1;
  for (int pitch = S.w; pitch < S.w + 32; ++pitch) {
    long total = 0;
    for (int rank = 0; rank < team; ++rank) {
      const int qb = (int)((int64_t)P.cells * rank / team);
      const int qe = (int)((int64_t)P.cells * (rank + 1) / team);
      const int items = (qe - qb) * blk;
      for (int w0 = 0; w0 < items; w0 += 32) {
        int addr[32], n = 0;
        for (int it = w0; it < std::min(items, w0 + 32); ++it) {
          const int pp = (qb + it / blk) % phw, t = it % blk;
          const int r = (pp / P.w) * P.py + t / P.px, c = (pp % P.w) * P.px + t % P.px;
          addr[n++] = r * L.ty * pitch + c * L.tx;
        }
        int worst = 0;
        for (int bank = 0; bank < 32; ++bank) {
          int distinct = 0;
          for (int i = 0; i < n; ++i) {
            if (addr[i] % 32 != bank) continue;
            bool seen = false;
            for (int j = 0; j < i; ++j) seen = seen || addr[j] == addr[i];
            distinct += seen ? 0 : 1;
          }
          worst = std::max(worst, distinct);
        }
        total += worst;
      }
    }
    if (best < 0 || total < best) {
      best = total;
      best_pitch = pitch;
    }
  }
  return best_pitch;
}

// The whole device description of a net from its resolved layers -- pure
// host code (no CUDA calls), shared by ck_net_create and the spec generator.
int build_net_geometry(const ck_layer_desc* layers, int n_layers, NetGeo* geo,
                       std::vector<int>& tables, std::vector<double>& filt,
                       int64_t* n_params) {
  NetGeo& N = *geo;
  memset(&N, 0, sizeof(NetGeo));
  N.n_layers = n_layers;

  int64_t p_cursor = 0, a_cursor = 0, t_cursor = 0, f_cursor = 0;
  std::vector<int64_t> tab_off(n_layers, 0), filt_off(n_layers, 0);
  for (int k = 0; k < n_layers; ++k) {
    const ck_layer_desc& D = layers[k];
    LayerDev& L = N.L[k];
    L.kind = D.kind;
    L.maps = D.maps;
    L.h = D.height;
    L.w = D.width;
    if (D.kind == CK_LAYER_FC) L.h = L.w = 1;
    L.cells = L.maps * L.h * L.w;
    if (L.maps < 1 || L.h < 1 || L.w < 1) {
      return set_error(CK_E_GEOMETRY, "layer " + std::to_string(k) + ": size below 1");
    }
    if (k > 0) {
      const LayerDev& S = N.L[k - 1];
      L.src_maps = S.maps;
      L.src_h = S.h;
      L.src_w = S.w;
      L.src_cells = S.cells;
    }
    L.has_delta = (D.kind == CK_LAYER_CONV || D.kind == CK_LAYER_POOL || D.kind == CK_LAYER_FC);
    L.y_off = a_cursor;
    a_cursor = align32(a_cursor + L.cells);
    if (D.kind == CK_LAYER_CONV || D.kind == CK_LAYER_FC) {
      L.a_off = a_cursor;
      a_cursor = align32(a_cursor + L.cells);
    }
    if (L.has_delta) {
      L.d_off = a_cursor;
      a_cursor = align32(a_cursor + L.cells);
    }
    if (D.kind == CK_LAYER_POOL) {
      L.arg_off = a_cursor;
      a_cursor = align32(a_cursor + L.cells);
      if (k > 0 && N.L[k - 1].kind == L_CONV) {   // compact winner data for the sparse backward
        LayerDev& C = N.L[k - 1];
        C.pool_above = C.has_delta;
        // weight_grad lane layout: tap-major (lanes = taps x groups walking
        // the winners) or winner-major (lanes walk winners, per-tap partials
        // + xor trees); pick the cheaper one for this geometry
        // weight gradients: each pair's sum over its winners is cut into
        // wg_split chunks of <= 32 winners (one lane group each, combined in
        // chunk order: a geometry constant, so results never depend on the team)
        const int kk = C.kx * C.ky, phw = D.width * D.height;
        C.wg_split = std::max(1, std::min(16, (phw + 31) / 32));
        // pull streams: lane groups (one winner each, lane = tap) x chunks of
        // the backward list, <= 16 f64 copies of a source map in shared memory
        C.pull_g = kk >= 32 ? 1 : std::min(32 / kk, phw);
        C.pull_ch = std::max(1, 16 / C.pull_g);
        // the pull as a bit-exact gather (conv_pull_gather); CKB200_PULL=scatter: A/B
        {
          const char* pm = getenv("CKB200_PULL");
          const int prm = ((C.ky - 1) / C.ty + D.py - 1) / D.py + 1;
          const int pcm = ((C.kx - 1) / C.tx + D.px - 1) / D.px + 1;
          // staged: every dest map's winners + one source map's backward
          // kernels at a time (re-checked with the tables below); else the scatter
          C.pullg = (pm && strcmp(pm, "scatter") == 0) || prm > 5 || pcm > 5 ? 0 : 1;
        }
        const int src_cells = N.L[k - 2].h * N.L[k - 2].w;
        while (C.pull_ch > 1 && C.pull_ch * C.pull_g * src_cells * 2 > kTeamStageFloats / 2)
          --C.pull_ch;
        L.wrc_off = a_cursor;
        a_cursor = align32(a_cursor + L.cells);
        L.wd_off = a_cursor;
        a_cursor = align32(a_cursor + L.cells);
      }
    }
    std::string where = "layer " + std::to_string(k) + ": ";
    switch (D.kind) {
      case CK_LAYER_INPUT:
        if (k != 0) { return set_error(CK_E_CONFIG, where + "input must be first"); }
        N.in_cells = L.cells;
        break;
      case CK_LAYER_IMGPROC:
        if (k != 1 || D.n_filters < 1 || !D.filter_coeffs || D.filter_h < 1 || D.filter_w < 1 ||
            D.maps != N.L[0].maps * (1 + D.n_filters) || D.width != N.L[0].w ||
            D.height != N.L[0].h) {
          return set_error(CK_E_CONFIG, where + "bad image-processing layer");
        }
        L.n_filt = D.n_filters;
        L.fh = D.filter_h;
        L.fw = D.filter_w;
        filt_off[k] = f_cursor;
        f_cursor += (int64_t)D.n_filters * D.filter_h * D.filter_w;
        break;
      case CK_LAYER_CONV: {
        const LayerDev& S = N.L[k - 1];
        if (D.kx < 1 || D.ky < 1 || D.sx < 0 || D.sy < 0 ||
            (L.h - 1) * (D.sy + 1) + D.ky > S.h || (L.w - 1) * (D.sx + 1) + D.kx > S.w) {
          return set_error(CK_E_GEOMETRY, where + "conv geometry does not fit its input");
        }
        if (!D.fwd_offsets || !D.fwd_srcs || !D.fwd_widx || !D.bias_offset ||
            D.arena_size != D.n_pairs * D.kx * D.ky + D.maps) {
          return set_error(CK_E_CONFIG, where + "incomplete connection table");
        }
        L.kx = D.kx; L.ky = D.ky; L.tx = D.sx + 1; L.ty = D.sy + 1;
        L.n_pairs = D.n_pairs;
        L.p_off = p_cursor;
        L.n_par = D.arena_size;
        p_cursor += D.arena_size;
        tab_off[k] = t_cursor;
        // fwd_off(maps+1) fwd_src fwd_widx bias(maps) bwd_off(src+1) bwd_dst bwd_widx pair_dst
        t_cursor += (L.maps + 1) + 2 * (int64_t)D.n_pairs + L.maps + (S.maps + 1) +
                    2 * (int64_t)D.n_pairs + D.n_pairs;
        break;
      }
      case CK_LAYER_POOL: {
        const LayerDev& S = N.L[k - 1];
        if (D.px < 1 || D.py < 1 || L.maps != S.maps || L.w != S.w / D.px || L.h != S.h / D.py) {
          return set_error(CK_E_GEOMETRY, where + "pool geometry does not match its input");
        }
        L.px = D.px; L.py = D.py;
        break;
      }
      case CK_LAYER_FC: {
        const LayerDev& S = N.L[k - 1];
        L.p_off = p_cursor;
        L.b_off = p_cursor + (int64_t)S.cells * L.cells;
        L.n_par = (int64_t)S.cells * L.cells + L.cells;
        p_cursor += L.n_par;
        break;
      }
      default:
        return set_error(CK_E_CONFIG, where + "unknown layer kind");
    }
  }
  for (int k = 0; k < n_layers; ++k)   // work splits use 32-bit (n * team size) products
    if (N.L[k].cells > (1 << 22) || N.L[k].n_par > (1 << 22)) {
      return set_error(CK_E_CONFIG, "layer " + std::to_string(k) + ": more than 4M cells/params");
    }
  N.n_classes = N.L[n_layers - 1].cells;
  if (N.n_classes > kScratchDoubles) {
    return set_error(CK_E_CONFIG, "too many output classes");
  }
  // pre-pitched copies of pool outputs a conv+pool consumes (conv_pool_fwd)
  for (int k = 2; k + 1 < n_layers && !getenv("CKB200_NO_PITCH"); ++k) {   // A/B switch
    LayerDev& S = N.L[k - 1];
    if (N.L[k].kind != L_CONV || N.L[k + 1].kind != L_POOL || S.kind != L_POOL) continue;
    // only when the consumer stages the layer whole or in source passes
    // (full tables, conv_pool_fwd_passes) -- not for per-map slots
    const bool whole = S.cells <= kTeamStageFloats / 2;
    bool full_table = layers[k].n_pairs == N.L[k].maps * S.maps;
    for (int p = 0; full_table && p < layers[k].n_pairs; ++p)
      full_table = layers[k].fwd_srcs[p] == p % S.maps;
    if (!whole && !full_table) continue;
    const int pitch = choose_src_pitch(N.L[k], S, N.L[k + 1]);
    if (pitch <= S.w || (whole && S.maps * S.h * pitch > kTeamStageFloats / 8 * 5)) continue;
    N.L[k].spitch = pitch;
    S.ypitch = pitch;
    S.yp_off = a_cursor;
    a_cursor = align32(a_cursor + (int64_t)S.maps * S.h * pitch);
  }
  N.act_size = a_cursor;
  *n_params = p_cursor;

  // host staging of the int32 tables
  tables.assign(std::max<int64_t>(t_cursor, 1), 0);
  for (int k = 0; k < n_layers; ++k) {
    if (layers[k].kind != CK_LAYER_CONV) continue;
    const ck_layer_desc& D = layers[k];
    const LayerDev& L = N.L[k];
    const int n_src = N.L[k - 1].maps;
    int* t = tables.data() + tab_off[k];
    int* fwd_off = t;           t += L.maps + 1;
    int* fwd_src = t;           t += D.n_pairs;
    int* fwd_widx = t;          t += D.n_pairs;
    int* bias = t;              t += L.maps;
    int* bwd_off = t;           t += n_src + 1;
    int* bwd_dst = t;           t += D.n_pairs;
    int* bwd_widx = t;          t += D.n_pairs;
    int* pair_dst = t;
    for (int d = 0; d <= L.maps; ++d) fwd_off[d] = (int)D.fwd_offsets[d];
    if (fwd_off[L.maps] != D.n_pairs) {
      return set_error(CK_E_CONFIG, "layer " + std::to_string(k) + ": CSR size mismatch");
    }
    std::vector<int> count(n_src, 0);
    for (int p = 0; p < D.n_pairs; ++p) {
      const int64_t s = D.fwd_srcs[p];
      if (s < 0 || s >= n_src || D.fwd_widx[p] < 0 ||
          D.fwd_widx[p] + D.kx * D.ky > D.arena_size) {
        return set_error(CK_E_CONFIG, "layer " + std::to_string(k) + ": table entry out of range");
      }
      fwd_src[p] = (int)s;
      fwd_widx[p] = (int)D.fwd_widx[p];
      count[s]++;
    }
    // The kernels rely on the reference's arena tiling (topology.py:82-96):
    // per dest map, its kx*ky blocks back to back in row order, then the bias.
    int cursor = 0;
    for (int d = 0; d < L.maps; ++d) {
      bias[d] = (int)D.bias_offset[d];
      for (int p = fwd_off[d]; p < fwd_off[d + 1]; ++p) {
        pair_dst[p] = d;
        if (fwd_widx[p] != cursor) {
          return set_error(CK_E_CONFIG, "layer " + std::to_string(k) +
                                            ": arena is not tiled like ConnectionTable");
        }
        cursor += D.kx * D.ky;
      }
      if (bias[d] != cursor) {
        return set_error(CK_E_CONFIG, "layer " + std::to_string(k) + ": bias slot out of place");
      }
      cursor += 1;
      N.L[k].max_fan_in = std::max(N.L[k].max_fan_in, fwd_off[d + 1] - fwd_off[d]);
    }
    // full table in ConnectionTable order: entries become arithmetic on device
    {
      bool full = D.n_pairs == L.maps * n_src;
      for (int p = 0; full && p < D.n_pairs; ++p)
        full = fwd_src[p] == p % n_src && pair_dst[p] == p / n_src;
      N.L[k].full = full ? 1 : 0;
    }
    // gather pull: measured faster than the stream scatter for very wide
    // backward lists (C4': 300 dests per source, 399 -> 156 us per image in
    // the pull phase) and for 2x2 kernels (C4 conv2: 28 -> 25 us); C1-C3
    // (5x5) are faster with the scatter -- and it needs all winners + the
    // widest source's backward kernels staged
    if (k + 1 < n_layers && N.L[k].pullg) {
      const int phw = N.L[k + 1].h * N.L[k + 1].w;
      const int widest = *std::max_element(count.begin(), count.end());
      const char* pm = getenv("CKB200_PULL");
      const bool forced = pm && strcmp(pm, "gather") == 0;
      if ((widest < 128 && D.kx * D.ky > 4 && !forced) ||
          2 * ((L.maps * phw + 3) & ~3) + widest * (D.kx * D.ky + 1) + 4 > kTeamStageFloats)
        N.L[k].pullg = 0;
    }
    // backward CSR = exact transpose, destinations ascending (topology.invert_table)
    bwd_off[0] = 0;
    for (int s = 0; s < n_src; ++s) bwd_off[s + 1] = bwd_off[s] + count[s];
    std::vector<int> fill(bwd_off, bwd_off + n_src);
    for (int d = 0; d < L.maps; ++d)
      for (int p = fwd_off[d]; p < fwd_off[d + 1]; ++p) {
        const int s = fwd_src[p];
        bwd_dst[fill[s]] = d;
        bwd_widx[fill[s]] = fwd_widx[p];
        fill[s]++;
      }
  }
  filt.assign(std::max<int64_t>(f_cursor, 1), 0.0);
  for (int k = 0; k < n_layers; ++k)
    if (layers[k].kind == CK_LAYER_IMGPROC)
      memcpy(filt.data() + filt_off[k], layers[k].filter_coeffs,
             sizeof(double) * layers[k].n_filters * layers[k].filter_h * layers[k].filter_w);

  for (int k = 0; k < n_layers; ++k) {   // table / filter offsets (LayerDev::o_*)
    LayerDev& L = N.L[k];
    if (L.kind == L_CONV) {
      int t = (int)tab_off[k];
      const int n_src = N.L[k - 1].maps;
      L.o_fwd_off = t;   t += L.maps + 1;
      L.o_fwd_src = t;   t += L.n_pairs;
      L.o_fwd_widx = t;  t += L.n_pairs;
      L.o_bias_off = t;  t += L.maps;
      L.o_bwd_off = t;   t += n_src + 1;
      L.o_bwd_dst = t;   t += L.n_pairs;
      L.o_bwd_widx = t;  t += L.n_pairs;
      L.o_pair_dst = t;
    }
    if (L.kind == L_IMGPROC) L.o_filt = (int)filt_off[k];
  }
  bool ok = true;
  build_programs(N, &ok);
  if (!ok) return set_error(CK_E_CONFIG, "network too deep for the phase program");
  return CK_OK;

}

// ---- specialised kernels: registry, geometry matching, source printer

bool layer_equal(const LayerDev& a, const LayerDev& b) {
#define CK_EQ(t, f) if (a.f != b.f) return false;
  CK_LAYER_FIELDS(CK_EQ)
#undef CK_EQ
  return true;
}

bool geo_equal(const NetGeo& a, const NetGeo& b) {
  if (a.n_layers != b.n_layers || a.n_classes != b.n_classes || a.in_cells != b.in_cells ||
      a.act_size != b.act_size)
    return false;
  for (int k = 0; k < a.n_layers; ++k)
    if (!layer_equal(a.L[k], b.L[k])) return false;
  for (int p = 0; p < N_PROGS; ++p) {
    const Program& x = a.prog[p];
    const Program& y = b.prog[p];
    if (x.n_phases != y.n_phases) return false;
    for (int i = 0; i <= x.n_phases; ++i)
      if (x.begin[i] != y.begin[i]) return false;
    for (int o = 0; o < x.begin[x.n_phases]; ++o)
      if (x.ops[o].kind != y.ops[o].kind || x.ops[o].layer != y.ops[o].layer ||
          x.ops[o].flags != y.ops[o].flags)
        return false;
  }
  return true;
}

int find_spec(const NetGeo& g) {
  int n = 0;
  const SpecEntry* t = spec_table(&n);
  for (int i = 0; i < n; ++i)
    if (geo_equal(g, t[i].geo)) return i;
  return -1;
}

// C++ source of `struct <name>` whose constexpr geo() equals g.
std::string spec_source(const NetGeo& g, const char* name) {
  std::string o;
  char b[256];
  o += "struct " + std::string(name) + " {\n";
  o += "  __host__ __device__ static constexpr NetGeo geo() {\n    NetGeo g{};\n";
  snprintf(b, sizeof b, "    g.n_layers = %d; g.n_classes = %d; g.in_cells = %d; g.act_size = %lldLL;\n",
           g.n_layers, g.n_classes, g.in_cells, (long long)g.act_size);
  o += b;
  for (int k = 0; k < g.n_layers; ++k) {
    const LayerDev& L = g.L[k];
    o += "    g.L[" + std::to_string(k) + "] = LayerDev{";
    bool first = true;
#define CK_PR(t, f)                                            \
  o += first ? "" : ", ";                                       \
  first = false;                                                \
  o += std::to_string((long long)L.f) + (sizeof(t) == 8 ? "LL" : "");
    CK_LAYER_FIELDS(CK_PR)
#undef CK_PR
    o += "};\n";
  }
  for (int p = 0; p < N_PROGS; ++p) {
    const Program& P = g.prog[p];
    snprintf(b, sizeof b, "    g.prog[%d].n_phases = %d;\n", p, P.n_phases);
    o += b;
    for (int i = 0; i <= P.n_phases; ++i) {
      snprintf(b, sizeof b, "    g.prog[%d].begin[%d] = %d;\n", p, i, P.begin[i]);
      o += b;
    }
    for (int i = 0; i < P.begin[P.n_phases]; ++i) {
      snprintf(b, sizeof b, "    g.prog[%d].ops[%d] = Op{%d, %d, %d, 0};\n", p, i, P.ops[i].kind,
               P.ops[i].layer, P.ops[i].flags);
      o += b;
    }
  }
  o += "    return g;\n  }\n";
  o += "  __device__ static const NetGeo& dev();\n};\n";
  // an immutable device object: loads from it fold to immediates
  o += "__device__ constexpr NetGeo kGeo_" + std::string(name) + " = " + name + "::geo();\n";
  o += "__device__ inline const NetGeo& " + std::string(name) + "::dev() { return kGeo_" + name +
       "; }\n";
  return o;
}

// Batched image-processing prepass for training launches: the contrast layer
// depends on the input image only, so instead of a team phase per image (all
// CTAs, then a barrier) every visited image's layer is computed up front by
// this kernel -- kPreSplit CTAs per image, the image staged in shared memory,
// contrast_cell's arithmetic (the per-image op's bits exactly).  Output: the
// layer's y (original channels, then the responses) of visit t at out + t *
// L.cells; the training kernel reads it (Job::pre) and skips phase 0.
constexpr int kPreSplit = 4;
__global__ void __launch_bounds__(256)
contrast_pre_kernel(LayerDev L, const double* __restrict__ filt, const uint8_t* images,
                    const float* lut, const int32_t* order, int64_t n, int in_cells,
                    float* out) {
  extern __shared__ float img[];
  const int64_t t = blockIdx.x / kPreSplit;
  const int part = blockIdx.x % kPreSplit;
  if (t >= n) return;
  const int64_t im = order ? (int64_t)__ldg(order + t) : t;
  if (lut)
    for (int i = threadIdx.x; i < in_cells; i += blockDim.x)
      img[i] = __ldg(lut + __ldg(images + im * in_cells + i));
  else
    for (int i = threadIdx.x; i < in_cells; i += blockDim.x)
      img[i] = __ldg(reinterpret_cast<const float*>(images) + im * in_cells + i);
  __syncthreads();
  float* o = out + t * (int64_t)L.cells;
  const int hw = L.h * L.w, C = L.src_maps, n_resp = L.cells - C * hw;
  if (part == 0)
    for (int i = threadIdx.x; i < C * hw; i += blockDim.x) o[i] = img[i];
  const int lane = threadIdx.x & 31, sub = threadIdx.x % kImgLanes;
  const unsigned gmask = ((1u << kImgLanes) - 1) << (lane & ~(kImgLanes - 1));
  const int chunk = (n_resp + kPreSplit - 1) / kPreSplit;
  const int r1 = min(n_resp, (part + 1) * chunk);
  for (int r = part * chunk + threadIdx.x / kImgLanes; r < r1; r += blockDim.x / kImgLanes) {
    const double acc = contrast_cell(L, img, filt + L.o_filt, C * hw + r, sub, gmask);
    if (sub == 0) o[C * hw + r] = (float)acc;
  }
}

// The same layer, same bits, laid out for the f64 pipe (contrast_strips,
// ck_engine.cuh): one CTA per (visit, channel), the channel staged once as
// f64 with its replicated border.
constexpr int kPreThreads = 288;

__global__ void __launch_bounds__(kPreThreads)
contrast_pre_strip_kernel(LayerDev L, const double* __restrict__ filt, const uint8_t* images,
                          const float* lut, const int32_t* order, int64_t n, int in_cells,
                          float* out) {
  extern __shared__ double dsm[];
  const int C = L.src_maps, H = L.h, W = L.w, hw = H * W;
  const int fh = L.fh, fw = L.fw, cy = fh / 2, cx = fw / 2;
  const int F = (L.cells - C * hw) / (C * hw);
  const int PW = strip_pitch(L), PH = H + fh - 1;
  double* win = dsm;                          // PH x PW, replicated border
  double* kf = dsm + (size_t)PH * PW;         // F x fh x fw
  const int64_t t = blockIdx.x / C;
  const int c = blockIdx.x % C;
  if (t >= n) return;
  const int64_t im = order ? (int64_t)__ldg(order + t) : t;
  const int64_t src0 = im * in_cells + (int64_t)c * hw;
  float* o = out + t * (int64_t)L.cells;
  for (int i = threadIdx.x; i < PH * PW; i += blockDim.x) {
    const int r = min(max(i / PW - cy, 0), H - 1), q = min(max(i % PW - cx, 0), W - 1);
    const float v = lut ? __ldg(lut + __ldg(images + src0 + r * W + q))
                        : __ldg(reinterpret_cast<const float*>(images) + src0 + r * W + q);
    win[i] = (double)v;
    if (i / PW >= cy && i / PW < cy + H && i % PW >= cx && i % PW < cx + W)
      o[c * hw + (i / PW - cy) * W + (i % PW - cx)] = v;   // the original channel
  }
  for (int i = threadIdx.x; i < F * fh * fw; i += blockDim.x) kf[i] = __ldg(filt + L.o_filt + i);
  __syncthreads();
  contrast_strips(L, win, kf, c, o);
}

// The prepass for a training launch over `n` visits (nullptr in *pre when the
// net has no image-processing layer, or CKB200_NO_PRE is set: A/B switch).
int run_prepass(ck_net* net, const uint8_t* images, const float* lut, const int32_t* order,
                int64_t n, cudaStream_t st, const float** pre) {
  *pre = nullptr;
  const NetGeo& N = net->h;
  if (N.n_layers < 2 || N.L[1].kind != L_IMGPROC || getenv("CKB200_NO_PRE")) return CK_OK;
  const int64_t need = n * (int64_t)N.L[1].cells;
  if (need > net->pre_cap) {
    CK_CUDA_TRY(cudaStreamSynchronize(st));
    cudaFree(net->d_pre);
    net->d_pre = nullptr;
    net->pre_cap = 0;
    CK_CUDA_TRY(cudaMalloc((void**)&net->d_pre, sizeof(float) * need));
    net->pre_cap = need;
  }
  static bool attr = false;
  if (!attr) {
    CK_CUDA_TRY(cudaFuncSetAttribute(contrast_pre_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK_CUDA_TRY(cudaFuncSetAttribute(contrast_pre_strip_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  const LayerDev& I = N.L[1];
  const int n_filt = (I.cells - I.src_maps * I.h * I.w) / (I.src_maps * I.h * I.w);
  const size_t strip_smem = sizeof(double) * ((size_t)(I.h + I.fh - 1) * strip_pitch(I) +
                                              (size_t)n_filt * I.fh * I.fw);
  if (strip_smem <= 200 * 1024 && !getenv("CKB200_PRE_LANES")) {
    contrast_pre_strip_kernel<<<(unsigned)(n * I.src_maps), kPreThreads, strip_smem, st>>>(
        I, net->d_filters, images, lut, order, n, N.in_cells, net->d_pre);
  } else {
    const size_t smem = sizeof(float) * N.in_cells;
    CK_CHECK(smem <= 200 * 1024, CK_E_DIMENSION, "input image too large for the prepass");
    contrast_pre_kernel<<<(unsigned)(n * kPreSplit), 256, smem, st>>>(
        N.L[1], net->d_filters, images, lut, order, n, N.in_cells, net->d_pre);
  }
  count_launch();
  CK_CUDA_TRY(cudaGetLastError());
  *pre = net->d_pre;
  return CK_OK;
}

}  // namespace

extern "C" {

int ck_net_create(const ck_layer_desc* layers, int n_layers, int device, ck_net** out) {
  CK_CHECK(layers && out, CK_E_CONFIG, "null argument");
  CK_CHECK(n_layers >= 2 && n_layers <= kMaxLayers, CK_E_CONFIG, "layer count out of range");
  CK_CHECK(layers[0].kind == CK_LAYER_INPUT, CK_E_CONFIG, "first layer must be the input");
  CK_CHECK(layers[n_layers - 1].kind == CK_LAYER_FC, CK_E_CONFIG,
           "last layer must be fully connected (output)");
  CK_CUDA_TRY(cudaSetDevice(device));

  ck_net* net = new ck_net();
  net->device = device;
  std::vector<int> tables;
  std::vector<double> filt;
  {
    const int rc = build_net_geometry(layers, n_layers, &net->h, tables, filt, &net->n_params);
    if (rc) {
      delete net;
      return rc;
    }
  }
  NetGeo& N = net->h;
  const int64_t p_cursor = net->n_params;
  net->spec = find_spec(N);
  if (getenv("CKB200_NO_SPEC")) net->use_spec = 0;   // A/B switch for measurements
  auto fail = [&](int rc) {
    ck_net_destroy(net);
    return rc;
  };
  cudaError_t e;
#define CK_ALLOC(ptr, bytes)                                        \
  e = cudaMalloc((void**)&(ptr), (bytes));                          \
  if (e != cudaSuccess) return fail(cuda_status(e, "cudaMalloc"));
  CK_ALLOC(net->d_desc, sizeof(NetGeo));
  CK_ALLOC(net->d_params, sizeof(float) * std::max<int64_t>(p_cursor, 1));
  CK_ALLOC(net->d_grads, sizeof(float) * std::max<int64_t>(p_cursor, 1));
  CK_ALLOC(net->d_act, sizeof(float) * N.act_size);
  CK_ALLOC(net->d_tables, sizeof(int) * tables.size());
  CK_ALLOC(net->d_filters, sizeof(double) * filt.size());
  CK_ALLOC(net->d_bar, 2 * sizeof(unsigned));
  CK_ALLOC(net->d_targets, sizeof(double) * N.n_classes);
  CK_ALLOC(net->d_loss, sizeof(double) * 2);
#undef CK_ALLOC
  e = cudaStreamCreateWithFlags(&net->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return fail(cuda_status(e, "cudaStreamCreate"));

  net->ptr.params = net->d_params;
  net->ptr.grads = net->d_grads;
  net->ptr.act = net->d_act;
  net->ptr.bar = net->d_bar;
  net->ptr.tables = net->d_tables;
  net->ptr.filt = net->d_filters;
  e = cudaMemcpy(net->d_tables, tables.data(), sizeof(int) * tables.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return fail(cuda_status(e, "upload tables"));
  e = cudaMemcpy(net->d_filters, filt.data(), sizeof(double) * filt.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return fail(cuda_status(e, "upload filters"));
  e = cudaMemcpy(net->d_desc, &N, sizeof(NetGeo), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return fail(cuda_status(e, "upload descriptor"));
  e = cudaMemset(net->d_bar, 0, 2 * sizeof(unsigned));
  if (e != cudaSuccess) return fail(cuda_status(e, "zero barrier"));
  e = cudaMemset(net->d_act, 0, sizeof(float) * N.act_size);
  if (e != cudaSuccess) return fail(cuda_status(e, "zero activations"));
  e = cudaMemset(net->d_grads, 0, sizeof(float) * std::max<int64_t>(p_cursor, 1));
  if (e != cudaSuccess) return fail(cuda_status(e, "zero grads"));
  *out = net;
  return CK_OK;
}

int ck_net_destroy(ck_net* net) {
  if (!net) return CK_OK;
  cudaSetDevice(net->device);
  if (net->stream) cudaStreamDestroy(net->stream);
  cudaFree(net->d_desc);
  cudaFree(net->d_params);
  cudaFree(net->d_grads);
  cudaFree(net->d_act);
  cudaFree(net->d_tables);
  cudaFree(net->d_filters);
  cudaFree(net->d_bar);
  cudaFree(net->d_targets);
  cudaFree(net->d_loss);
  cudaFree(net->d_eval);
  cudaFree(net->d_pre);
  delete net;
  return CK_OK;
}

int ck_net_set_team(ck_net* net, int kind, int ctas, int threads) {
  CK_CHECK(net, CK_E_CONFIG, "null net");
  if (kind == CK_TEAM_AUTO) {
    net->team_kind = CK_TEAM_AUTO;
    net->team_ctas = 0;
    net->threads = 512;
    return CK_OK;
  }
  CK_CHECK(kind == CK_TEAM_CLUSTER || kind == CK_TEAM_GRID, CK_E_CONFIG, "unknown team kind");
  CK_CHECK(threads >= 32 && threads <= 512 && threads % 32 == 0, CK_E_CONFIG,
           "threads must be a multiple of 32 in [32, 512]");
  CK_CHECK(ctas >= 1 && ctas <= 1024 && (kind == CK_TEAM_GRID || ctas <= 16), CK_E_CONFIG,
           "cluster teams hold 1..16 CTAs, grid teams 1..1024");
  net->team_kind = kind;
  net->team_ctas = ctas;
  net->threads = threads;
  return CK_OK;
}

int ck_net_get_team(const ck_net* net, int* kind, int* ctas, int* threads) {
  CK_CHECK(net && kind && ctas && threads, CK_E_CONFIG, "null argument");
  const TeamShape t = resolve_team(net, 1);   // what a single-net launch uses
  *kind = t.kind;
  *ctas = t.ctas;
  *threads = t.threads;
  return CK_OK;
}

int ck_net_num_params(const ck_net* net, int64_t* n) {
  CK_CHECK(net && n, CK_E_CONFIG, "null argument");
  *n = net->n_params;
  return CK_OK;
}

int ck_net_set_params(ck_net* net, const float* host, int64_t n) {
  CK_CHECK(net && host, CK_E_CONFIG, "null argument");
  CK_CHECK(n == net->n_params, CK_E_DIMENSION, "parameter count mismatch");
  { const int q = quiesce(net); if (q) return q; }
  CK_CUDA_TRY(cudaSetDevice(net->device));
  CK_CUDA_TRY(cudaMemcpy(net->d_params, host, sizeof(float) * n, cudaMemcpyHostToDevice));
  return CK_OK;
}

int ck_net_device_params(const ck_net* net, const float** params) {
  CK_CHECK(net && params, CK_E_CONFIG, "null argument");
  *params = net->d_params;
  return CK_OK;
}

int ck_net_get_params(ck_net* net, float* host, int64_t n) {
  CK_CHECK(net && host, CK_E_CONFIG, "null argument");
  CK_CHECK(n == net->n_params, CK_E_DIMENSION, "parameter count mismatch");
  { const int q = quiesce(net); if (q) return q; }
  CK_CUDA_TRY(cudaSetDevice(net->device));
  CK_CUDA_TRY(cudaMemcpy(host, net->d_params, sizeof(float) * n, cudaMemcpyDeviceToHost));
  return CK_OK;
}

static int stage_input(ck_net* net, const float* x) {
  const LayerDev& I = net->h.L[0];
  CK_CUDA_TRY(cudaMemcpyAsync(net->d_act + I.y_off, x, sizeof(float) * I.cells,
                              cudaMemcpyHostToDevice, net->stream));
  return CK_OK;
}

int ck_net_forward(ck_net* net, const float* x, float* y_out) {
  CK_CHECK(net && x, CK_E_CONFIG, "null argument");
  { const int q = quiesce(net); if (q) return q; }
  CK_CUDA_TRY(cudaSetDevice(net->device));
  int rc = stage_input(net, x);
  if (rc) return rc;
  Job job = empty_job(PROG_FORWARD);
  rc = run_single(net, job);
  if (rc) return rc;
  if (y_out) {
    const LayerDev& O = net->h.L[net->h.n_layers - 1];
    CK_CUDA_TRY(cudaMemcpy(y_out, net->d_act + O.y_off, sizeof(float) * O.cells,
                           cudaMemcpyDeviceToHost));
  }
  return CK_OK;
}

int ck_net_backward(ck_net* net, const double* targets) {
  CK_CHECK(net && targets, CK_E_CONFIG, "null argument");
  { const int q = quiesce(net); if (q) return q; }
  CK_CUDA_TRY(cudaSetDevice(net->device));
  CK_CUDA_TRY(cudaMemcpyAsync(net->d_targets, targets, sizeof(double) * net->h.n_classes,
                              cudaMemcpyHostToDevice, net->stream));
  Job job = empty_job(PROG_BACKWARD);
  job.targets = net->d_targets;
  return run_single(net, job);
}

int ck_net_apply_gradients(ck_net* net, double eta) {
  CK_CHECK(net, CK_E_CONFIG, "null net");
  CK_CHECK(eta > 0, CK_E_CONFIG, "learning rate must be > 0");
  { const int q = quiesce(net); if (q) return q; }
  Job job = empty_job(PROG_APPLY);
  job.eta_f = (float)eta;
  return run_single(net, job);
}

int ck_net_train_step(ck_net* net, const float* x, const double* targets, double eta,
                      double* loss) {
  CK_CHECK(net && x && targets, CK_E_CONFIG, "null argument");
  { const int q = quiesce(net); if (q) return q; }
  CK_CUDA_TRY(cudaSetDevice(net->device));
  int rc = stage_input(net, x);
  if (rc) return rc;
  CK_CUDA_TRY(cudaMemcpyAsync(net->d_targets, targets, sizeof(double) * net->h.n_classes,
                              cudaMemcpyHostToDevice, net->stream));
  // eta <= 0: forward + loss + gradients without an update (network.py:279-281)
  Job job = empty_job(eta > 0 ? PROG_TRAIN : PROG_BACKWARD);
  if (eta <= 0) {
    Job fwd = empty_job(PROG_FORWARD);
    rc = run_single(net, fwd);
    if (rc) return rc;
  }
  job.targets = net->d_targets;
  job.eta_f = (float)eta;
  rc = run_single(net, job);
  if (rc) return rc;
  if (loss) CK_CUDA_TRY(cudaMemcpy(loss, net->d_loss, sizeof(double), cudaMemcpyDeviceToHost));
  return CK_OK;
}

int ck_net_buffer_size(const ck_net* net, int layer, int which, int64_t* count) {
  CK_CHECK(net && count, CK_E_CONFIG, "null argument");
  CK_CHECK(layer >= 0 && layer < net->h.n_layers, CK_E_DIMENSION, "layer out of range");
  const LayerDev& L = net->h.L[layer];
  switch (which) {
    case CK_BUF_Y: *count = L.cells; return CK_OK;
    case CK_BUF_A:
      CK_CHECK(L.kind == L_CONV || L.kind == L_FC, CK_E_STATE, "layer has no pre-activations");
      *count = L.cells; return CK_OK;
    case CK_BUF_DELTA:
      CK_CHECK(L.has_delta, CK_E_STATE, "layer keeps no deltas");
      *count = L.cells; return CK_OK;
    case CK_BUF_ARG:
      CK_CHECK(L.kind == L_POOL, CK_E_STATE, "layer has no pool index");
      *count = L.cells; return CK_OK;
    case CK_BUF_GRAD:
      CK_CHECK(L.n_par > 0, CK_E_STATE, "layer has no parameters");
      *count = L.n_par; return CK_OK;
    default: return set_error(CK_E_CONFIG, "unknown buffer");
  }
}

int ck_net_read_buffer(ck_net* net, int layer, int which, void* host, int64_t count) {
  int64_t n = 0;
  int rc = ck_net_buffer_size(net, layer, which, &n);
  if (rc) return rc;
  { const int q = quiesce(net); if (q) return q; }
  CK_CHECK(host && count == n, CK_E_DIMENSION, "buffer size mismatch");
  CK_CUDA_TRY(cudaSetDevice(net->device));
  const LayerDev& L = net->h.L[layer];
  const void* src = nullptr;
  switch (which) {
    case CK_BUF_Y: src = net->d_act + L.y_off; break;
    case CK_BUF_A: src = net->d_act + L.a_off; break;
    case CK_BUF_DELTA: src = net->d_act + L.d_off; break;
    case CK_BUF_ARG: src = net->d_act + L.arg_off; break;
    case CK_BUF_GRAD: src = net->d_grads + L.p_off; break;
  }
  CK_CUDA_TRY(cudaMemcpy(host, src, 4 * n, cudaMemcpyDeviceToHost));
  return CK_OK;
}

int ck_committee_train_epoch(ck_net* const* nets, int n_nets, const uint8_t* images,
                             const float* lut, const int32_t* labels, const int32_t* order,
                             int64_t n, double eta, double* mean_losses, ck_stream_t stream) {
  CK_CHECK(nets && n_nets >= 1 && n_nets <= kMaxNetsPerLaunch, CK_E_CONFIG,
           "need 1..32 nets per launch (kMaxNetsPerLaunch; callers split larger committees)");
  CK_CHECK(images && labels, CK_E_CONFIG, "null dataset pointer");
  CK_CHECK(n >= 1, CK_E_CONFIG, "empty epoch");
  CK_CHECK(eta > 0, CK_E_CONFIG, "learning rate must be > 0");
  for (int i = 0; i < n_nets; ++i) {
    CK_CHECK(nets[i] && nets[i]->device == nets[0]->device, CK_E_CONFIG,
             "committee nets must live on one device");
    CK_CHECK(nets[i]->h.in_cells == nets[0]->h.in_cells, CK_E_DIMENSION,
             "committee nets must share the input geometry");
  }
  CK_CUDA_TRY(cudaSetDevice(nets[0]->device));
  double* d_tot = nullptr;
  CK_CUDA_TRY(cudaMallocAsync((void**)&d_tot, sizeof(double) * n_nets, (cudaStream_t)stream));
  Job job = empty_job(PROG_TRAIN);
  job.images = images;
  job.lut = lut;
  job.labels = labels;
  job.order = order;
  job.n = n;
  job.first = 0;
  job.eta_f = (float)eta;
  job.loss_total = d_tot;
  int rc = launch_teams(nets, n_nets, job, (cudaStream_t)stream);
  if (rc == CK_OK && mean_losses) {
    std::vector<double> tot(n_nets);
    cudaError_t e = cudaMemcpyAsync(tot.data(), d_tot, sizeof(double) * n_nets,
                                    cudaMemcpyDeviceToHost, (cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) rc = cuda_status(e, "read losses");
    for (int i = 0; i < n_nets && rc == CK_OK; ++i) mean_losses[i] = tot[i] / (double)n;
  }
  cudaFreeAsync(d_tot, (cudaStream_t)stream);
  return rc;
}

int ck_net_train_epoch(ck_net* net, const uint8_t* images, const float* lut,
                       const int32_t* labels, const int32_t* order, int64_t n, double eta,
                       double* losses, double* mean_loss, ck_stream_t stream) {
  CK_CHECK(net, CK_E_CONFIG, "null net");
  CK_CHECK(images && labels, CK_E_CONFIG, "null dataset pointer");
  CK_CHECK(n >= 1, CK_E_CONFIG, "empty epoch");
  CK_CHECK(eta > 0, CK_E_CONFIG, "learning rate must be > 0");
  CK_CUDA_TRY(cudaSetDevice(net->device));
  Job job = empty_job(PROG_TRAIN);
  job.images = images;
  job.lut = lut;
  job.labels = labels;
  job.order = order;
  job.n = n;
  job.eta_f = (float)eta;
  job.losses = losses;
  job.loss_total = net->d_loss;
  int rc = run_prepass(net, images, lut, order, n, (cudaStream_t)stream, &job.pre);
  if (rc) return rc;
  rc = launch_teams(&net, 1, job, (cudaStream_t)stream);
  if (rc) return rc;
  if (mean_loss) {
    double tot = 0;
    CK_CUDA_TRY(cudaMemcpyAsync(&tot, net->d_loss, sizeof(double), cudaMemcpyDeviceToHost,
                                (cudaStream_t)stream));
    CK_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    *mean_loss = tot / (double)n;
  }
  return CK_OK;
}

int ck_net_profile_epoch(ck_net* net, const uint8_t* images, const float* lut,
                         const int32_t* labels, const int32_t* order, int64_t n, double eta,
                         int64_t* phase_ns, int max_phases, int* n_phases) {
  CK_CHECK(net && images && labels && phase_ns && n_phases, CK_E_CONFIG, "null argument");
  CK_CHECK(n >= 1 && eta > 0, CK_E_CONFIG, "need images and a positive learning rate");
  CK_CUDA_TRY(cudaSetDevice(net->device));
  const int np = net->h.prog[PROG_TRAIN].n_phases;
  *n_phases = np;
  CK_CHECK(max_phases >= 2 * np, CK_E_DIMENSION, "phase buffer too small");
  const int ctas = resolve_team(net, 1).ctas;
  const int64_t stride = 1 + (int64_t)np * (1 + ctas);
  long long* d_prof = nullptr;
  CK_CUDA_TRY(cudaMalloc((void**)&d_prof, sizeof(long long) * n * stride));
  CK_CUDA_TRY(cudaMemset(d_prof, 0, sizeof(long long) * n * stride));
  Job job = empty_job(PROG_TRAIN);
  job.images = images;
  job.lut = lut;
  job.labels = labels;
  job.order = order;
  job.n = n;
  job.eta_f = (float)eta;
  job.loss_total = net->d_loss;
  job.prof = d_prof;
  job.prof_images = n;
  int rc = run_prepass(net, images, lut, order, n, net->stream, &job.pre);
  if (rc == CK_OK) rc = launch_teams(&net, 1, job, net->stream);
  std::vector<long long> h((size_t)(n * stride));
  if (rc == CK_OK) {
    cudaError_t e = cudaMemcpyAsync(h.data(), d_prof, sizeof(long long) * h.size(),
                                    cudaMemcpyDeviceToHost, net->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(net->stream);
    if (e != cudaSuccess) rc = cuda_status(e, "read phase profile");
  }
  cudaFree(d_prof);
  if (rc) return rc;
  // phase_ns[p]: slowest CTA's work (phase start -> its work end);
  // phase_ns[np + p]: barrier latency (slowest work end -> barrier exit)
  // (a phase skipped because its layers were precomputed -- Job::pre -- has
  // no records: it reads as zero work and the next phase starts at r[0])
  for (int p = 0; p < np; ++p) {
    long long work = 0, bar = 0;
    for (int64_t t = 0; t < n; ++t) {
      const long long* r = h.data() + t * stride;
      const long long* ph = r + 1 + p * (1 + ctas);
      if (ph[0] == 0) continue;
      long long start = r[0];
      for (int q = p - 1; q >= 0; --q)
        if (r[1 + q * (1 + ctas)] != 0) {
          start = r[1 + q * (1 + ctas)];
          break;
        }
      long long wmax = start;
      for (int c = 0; c < ctas; ++c) wmax = std::max(wmax, ph[1 + c]);
      work += wmax - start;
      bar += ph[0] - wmax;
    }
    phase_ns[p] = work / n;
    phase_ns[np + p] = bar / n;
  }
  return CK_OK;
}

int ck_net_spec_source(const ck_layer_desc* layers, int n_layers, const char* name, char* buf,
                       int64_t cap, int64_t* len) {
  CK_CHECK(layers && name && len, CK_E_CONFIG, "null argument");
  CK_CHECK(n_layers >= 2 && n_layers <= kMaxLayers, CK_E_CONFIG, "layer count out of range");
  NetGeo* g = new NetGeo();
  std::vector<int> tables;
  std::vector<double> filt;
  int64_t n_params = 0;
  const int rc = build_net_geometry(layers, n_layers, g, tables, filt, &n_params);
  if (rc) {
    delete g;
    return rc;
  }
  const std::string src = spec_source(*g, name);
  delete g;
  *len = (int64_t)src.size();
  if (buf && cap > (int64_t)src.size()) memcpy(buf, src.c_str(), src.size() + 1);
  return CK_OK;
}

int ck_net_set_specialized(ck_net* net, int enable) {
  CK_CHECK(net, CK_E_CONFIG, "null net");
  net->use_spec = enable ? 1 : 0;
  return CK_OK;
}

int ck_net_kernel_info(const ck_net* net, char* buf, int cap) {
  CK_CHECK(net && buf && cap > 0, CK_E_CONFIG, "null argument");
  int n = 0;
  const SpecEntry* t = spec_table(&n);
  if (net->spec >= 0 && net->use_spec)
    snprintf(buf, cap, "specialised:%s", t[net->spec].name);
  else
    snprintf(buf, cap, "generic");
  return CK_OK;
}

// Development aid (not in ckb200.h's stable surface): arm the sub-phase
// timers with a device buffer of >= 32 * n_phases int64 (NULL disarms).
int ck_debug_subprof(long long* dev_buf, int rank) {
  g_sub = dev_buf;
  g_sub_rank = rank;
  return CK_OK;
}

int ck_net_describe_program(const ck_net* net, int prog, char* buf, int cap) {
  CK_CHECK(net && buf && cap > 0, CK_E_CONFIG, "null argument");
  CK_CHECK(prog >= 0 && prog < N_PROGS, CK_E_CONFIG, "unknown program");
  static const char* names[] = {"load_input", "imgproc", "conv_fwd", "pool_fwd", "fc_fwd",
                                "zero_delta", "out_delta", "fc_bwd", "conv_bwd", "update",
                                "fc_out", "conv_pool"};
  const Program& P = net->h.prog[prog];
  std::string s;
  for (int ph = 0; ph < P.n_phases; ++ph) {
    s += "phase " + std::to_string(ph) + ":";
    for (int o = P.begin[ph]; o < P.begin[ph + 1]; ++o) {
      const Op& op = P.ops[o];
      s += std::string(" ") + names[op.kind] + "(L" + std::to_string(op.layer);
      if (op.flags & F_UPDATE) s += ",update";
      if (op.flags & F_PULL) s += ",pull";
      if (op.flags & F_ZERO_SELF) s += ",zero";
      s += ")";
    }
    s += "\n";
  }
  snprintf(buf, cap, "%s", s.c_str());
  return CK_OK;
}

int ck_net_eval(ck_net* net, const uint8_t* images, const float* lut, int64_t first,
                int64_t n, int32_t* pred, float* outputs, ck_stream_t stream) {
  CK_CHECK(net && images && pred, CK_E_CONFIG, "null argument");
  CK_CHECK(n >= 0 && first >= 0, CK_E_CONFIG, "bad image range");
  if (n == 0) return CK_OK;
  CK_CUDA_TRY(cudaSetDevice(net->device));
  int rc = configure_kernels();
  if (rc) return rc;
  int sms = 148;
  CK_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, net->device));
  const int floats = eval_floats_for(net->h);
  const int per_sm = floats == kEvalBigFloats ? 1 : 2;
  const int ctas = (int)std::min<int64_t>(n, (int64_t)sms * per_sm);
  if (ctas > net->eval_ctas) {
    CK_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    cudaFree(net->d_eval);
    net->d_eval = nullptr;
    net->eval_ctas = 0;
    CK_CUDA_TRY(cudaMalloc((void**)&net->d_eval, sizeof(float) * net->h.act_size * ctas));
    net->eval_ctas = ctas;
  }
  Job job = empty_job(PROG_EVAL);
  job.images = images;
  job.lut = lut;
  job.first = first;
  job.n = n;
  job.pred = pred;
  job.outputs = outputs;
  job.eval_scratch = net->d_eval;
  job.eval_floats = floats;
  if (net->spec >= 0 && net->use_spec) {
    int n_spec = 0;
    const void* k = spec_table(&n_spec)[net->spec].eval_kernel;
    static std::vector<const void*> configured;
    if (std::find(configured.begin(), configured.end(), k) == configured.end()) {
      CK_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)eval_smem_bytes()));
      configured.push_back(k);
    }
    const NetGeo* geo = net->d_desc;
    NetPtr R = net->ptr;
    void* args[] = {(void*)&geo, (void*)&R, (void*)&job};
    CK_CUDA_TRY(cudaLaunchKernel(k, dim3(ctas), dim3(256), args, eval_smem_bytes(floats),
                                 (cudaStream_t)stream));
  } else {
    net_eval_kernel<<<ctas, 256, eval_smem_bytes(floats), (cudaStream_t)stream>>>(
        net->d_desc, net->ptr, job);
  }
  count_launch();
  CK_CUDA_TRY(cudaGetLastError());
  return CK_OK;
}

}  // extern "C"
