// ck_kernels.cuh -- the device side of the network seam: teams and their
// barriers, the persistent training kernel (generic interpreter and the
// specialised template), batched evaluation.  Included by ck_net.cu (host
// runtime, generic kernels) and by the generated ck_spec_*.cu translation
// units (one specialised kernel each, compiled in parallel).
#pragma once
#include <stdint.h>

#include <type_traits>

#include "ck_engine.cuh"

#ifndef CK_TEAM_THREADS
#define CK_TEAM_THREADS 512
#endif

namespace ck {

constexpr int kMaxNetsPerLaunch = 32;
constexpr int kFuseHiddenMax = 4096;   // hidden FC width fused into OP_FC_OUT
constexpr int kScratchDoubles = 1024;  // output-layer scratch (n_classes <= 1024)

// Kernel argument: per net of the launch, its geometry (device copy, read by
// the generic kernels) and its memory.
struct NetRefs {
  const NetGeo* geo[kMaxNetsPerLaunch];
  NetPtr ptr[kMaxNetsPerLaunch];
};

// ---------------------------------------------------------------------------
// teams

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct ClusterTeam {
  __device__ static unsigned rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
  }
  __device__ static unsigned size() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
  }
  __device__ static unsigned index(int) {
    unsigned r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
  }
  __device__ static void sync(const NetPtr&, int, unsigned&) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
};

// Grid team barrier: a monotonic arrival counter (zeroed before each launch).
// Each CTA's thread 0 adds 1 with release semantics (cumulative over the
// CTA's writes, ordered before it by bar.sync) and polls with acquire until
// every CTA of this barrier generation has arrived.  No reset, no full
// fences.  The arrival returns the old count, so the last CTA to arrive
// skips the poll (tools/mb_barrier.cu: 2300 vs 2600 cycles per barrier with
// 2 KB of stores per CTA to release; ~1.1 us is two L2 round trips).
struct GridTeam {
  __device__ static unsigned rank(int ctas) { return blockIdx.x % ctas; }
  __device__ static unsigned index(int ctas) { return blockIdx.x / ctas; }
  __device__ static void sync(const NetPtr& R, int ctas, unsigned& target) {
    __syncthreads();
    if (threadIdx.x == 0) {
      target += (unsigned)ctas;
      unsigned old;
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(R.bar) : "memory");
      if (old + 1 != target) {
        while ((int)(ld_acquire(R.bar) - target) < 0) {
        }
      }
    }
    __syncthreads();
  }
};

// Point the team context at the current image (dataset bytes + LUT, f32
// dataset, or the host-staged input already in the activation arena).
__device__ __forceinline__ void set_input(const NetGeo& N, const Job& job, const Ctx& ctx,
                                          TeamCtx& tm) {
  tm.in_u8 = nullptr;
  tm.in_lut = nullptr;
  if (job.images && job.lut) {
    tm.in_u8 = job.images + ctx.img * (int64_t)N.in_cells;
    tm.in_lut = job.lut;
    tm.in_f32 = nullptr;
  } else if (job.images) {
    tm.in_f32 = reinterpret_cast<const float*>(job.images) + ctx.img * (int64_t)N.in_cells;
  } else {
    tm.in_f32 = ctx.act + N.L[0].y_off;
  }
}

// Copy a net descriptor into shared memory (descriptor reads then never
// touch L1/L2 inside the image loop).
__device__ __forceinline__ void load_desc(NetGeo* dst, const NetGeo* src) {
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(dst);
  for (int i = threadIdx.x; i < (int)(sizeof(NetGeo) / sizeof(int4)); i += blockDim.x) d[i] = s[i];
  __syncthreads();
}

// ---------------------------------------------------------------------------
// persistent training / single-step kernel: one team per net.

__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr size_t kDescBytes = (sizeof(NetGeo) + 15) & ~size_t(15);
constexpr size_t kScratchBytes = kScratchDoubles * sizeof(double);
constexpr int kTeamStageFloats = 48 * 1024;   // 192 KB staging per CTA
constexpr int kEvalStageFloats = 24 * 1024;   // 96 KB staging: 2 eval CTAs per SM
constexpr int kEvalBigFloats = 48 * 1024;     // 192 KB: 1 eval CTA per SM (wide nets)

// Where this CTA sits: its team (net) and rank.
template <class Team>
__device__ __forceinline__ void team_position(int ctas, unsigned& rank, unsigned& team,
                                              unsigned& tsize) {
  if constexpr (std::is_same<Team, ClusterTeam>::value) {
    rank = ClusterTeam::rank();
    tsize = ClusterTeam::size();
    team = ClusterTeam::index(ctas);
  } else {
    rank = GridTeam::rank(ctas);
    tsize = ctas;
    team = GridTeam::index(ctas);
  }
}

// The per-image loop of one team.  RunPhases(ph-loop body) is either the
// interpreted program (generic kernel) or a compile-time unrolled one
// (specialised kernels, ck_specs.cuh); everything else is shared.
template <class Team, class Phases>
__device__ __forceinline__ void team_loop(const NetGeo& N, const NetPtr& R, const Job& job,
                                          int ctas, unsigned rank, unsigned team,
                                          unsigned tsize, unsigned char* work, int n_phases,
                                          const Phases& phases) {
  double* scratch = reinterpret_cast<double*>(work);
  TeamCtx tm;
  tm.ph = 0;
  tm.sub = job.sub;
  tm.sub_rank = job.sub_rank;
  tm.rank = rank;
  tm.size = tsize;
  tm.gtid = rank * blockDim.x + threadIdx.x;
  tm.gsize = tsize * blockDim.x;
  tm.gwarp = tm.gtid >> 5;
  tm.gwarps = tm.gsize >> 5;
  tm.smem = reinterpret_cast<float*>(work + kScratchBytes);
  tm.smem_floats = kTeamStageFloats;
  Ctx ctx;
  ctx.act = R.act;
  ctx.loss = 0.0;
  double total = 0.0;
  // profile record per image: [start, then per phase: barrier exit (rank 0),
  // work end of every CTA (after its last warp)] -- globaltimer ns
  const int prof_stride = 1 + n_phases * (1 + (int)tsize);
  unsigned bar_target = 0;
  for (int64_t t = 0; t < job.n; ++t) {
    ctx.t = t;
    ctx.img = job.order ? (int64_t)__ldg(job.order + t) : job.first + t;
    ctx.label = job.labels ? __ldg(job.labels + ctx.img) : -1;
    set_input(N, job, ctx, tm);
    tm.pre = (job.pre && N.L[1].kind == L_IMGPROC) ? job.pre + ctx.t * (int64_t)N.L[1].cells
                                                   : nullptr;
    long long* prof = (job.prof && team == 0 && t < job.prof_images)
                          ? job.prof + t * prof_stride : nullptr;
    if (prof && rank == 0 && threadIdx.x == 0) prof[0] = globaltimer();
    auto after_phase = [&](int ph) {
      CK_SUBT(tm, 30);
      if (tm.sub && threadIdx.x == 0 && tm.rank == tm.sub_rank)
        tm.sub[ph * 32 + 29] = clock64();   // SM cycles at the same point (clock check)
      if (prof) {
        __syncthreads();
        if (threadIdx.x == 0) prof[1 + ph * (1 + tsize) + 1 + rank] = globaltimer();
      }
      Team::sync(R, ctas, bar_target);
      CK_SUBT(tm, 31);
      if (prof && rank == 0 && threadIdx.x == 0) prof[1 + ph * (1 + tsize)] = globaltimer();
    };
    phases(job, ctx, tm, scratch, after_phase);
    if (rank == 0 && threadIdx.x == 0 && job.prog != PROG_FORWARD && job.prog != PROG_APPLY) {
      total += ctx.loss;
      if (job.losses) job.losses[team * job.n + t] = ctx.loss;
    }
  }
  if (rank == 0 && threadIdx.x == 0 && job.loss_total) job.loss_total[team] = total;
}

// Interpreted phase program (any net, any program).
struct InterpPhases {
  const NetGeo& N;
  const NetPtr& R;
  template <class After>
  __device__ __forceinline__ void operator()(const Job& job, Ctx& ctx, TeamCtx& tm,
                                             double* scratch, After& after) const {
    const Program& P = N.prog[job.prog];
    const int ph0 = (tm.pre && phase0_input_only(P)) ? 1 : 0;   // precomputed input layers
    for (int ph = ph0; ph < P.n_phases; ++ph) {
      tm.ph = ph;
      CK_SUBT(tm, 0);
      run_phase(N, R, P, ph, job, ctx, tm, scratch);
      after(ph);
    }
  }
};

template <class Team>
__global__ void __launch_bounds__(CK_TEAM_THREADS, 1)
net_team_kernel(NetRefs nets, Job job, int ctas) {
  extern __shared__ __align__(16) unsigned char smem[];
  NetGeo& N = *reinterpret_cast<NetGeo*>(smem);
  unsigned rank, team, tsize;
  team_position<Team>(ctas, rank, team, tsize);
  if ((int)team >= job.n_nets) return;
  load_desc(&N, nets.geo[team]);
  const NetPtr R = nets.ptr[team];
  team_loop<Team>(N, R, job, ctas, rank, team, tsize, smem + kDescBytes,
                  N.prog[job.prog].n_phases, InterpPhases{N, R});
}

// ---------------------------------------------------------------------------
// Specialised training kernels.  ck_specs.inc (generated by
// tools/gen_specs.py from configs.ARCH through ck_net_spec_source) holds one
// struct per BASELINE net whose constexpr geo() is the exact NetGeo that
// build_net_geometry produces for it.  The kernel below walks PROG_TRAIN's
// phases and ops by compile-time recursion, so every layer index, size,
// offset and op choice is a constant: no interpreter, no runtime division,
// only the code the net needs.  Same ops, same arithmetic as the generic
// kernel -- results are bit-identical (tests/test_gpu_parity.py).

template <class Spec, int PROG, int PH, int O>
struct SpecOps {
  __device__ static __forceinline__ void run(const NetPtr& R, const Job& job, Ctx& ctx,
                                             const TeamCtx& tm, double* scratch) {
    if constexpr (O < Spec::geo().prog[PROG].begin[PH + 1]) {
      constexpr Op op = Spec::geo().prog[PROG].ops[O];
      run_op(Spec::dev(), R, op, job, ctx, tm, scratch);
      SpecOps<Spec, PROG, PH, O + 1>::run(R, job, ctx, tm, scratch);
    }
  }
};

template <class Spec, int PROG, int PH>
struct SpecPhase {
  template <class After>
  __device__ static __forceinline__ void run(const NetPtr& R, const Job& job, Ctx& ctx,
                                             TeamCtx& tm, double* scratch, After& after) {
    if constexpr (PH == 0 && phase0_input_only(Spec::geo().prog[PROG])) {
      if (tm.pre) {           // input layers precomputed by the batched prepass
        SpecPhase<Spec, PROG, 1>::run(R, job, ctx, tm, scratch, after);
        return;
      }
    }
    if constexpr (PH < Spec::geo().prog[PROG].n_phases) {
      tm.ph = PH;
      CK_SUBT(tm, 0);
      SpecOps<Spec, PROG, PH, Spec::geo().prog[PROG].begin[PH]>::run(R, job, ctx, tm, scratch);
      after(PH);
      SpecPhase<Spec, PROG, PH + 1>::run(R, job, ctx, tm, scratch, after);
    }
  }
};

template <class Spec>
struct SpecPhases {
  const NetPtr& R;
  template <class After>
  __device__ __forceinline__ void operator()(const Job& job, Ctx& ctx, TeamCtx& tm,
                                             double* scratch, After& after) const {
    SpecPhase<Spec, PROG_TRAIN, 0>::run(R, job, ctx, tm, scratch, after);
  }
};

template <class Spec>
struct SpecEval {
  const NetPtr& R;
  __device__ __forceinline__ void operator()(const Job& job, Ctx& ctx, TeamCtx& tm) const {
    auto sync = [](int) { __syncthreads(); };
    SpecPhase<Spec, PROG_EVAL, 0>::run(R, job, ctx, tm, nullptr, sync);
  }
};

// The specialised evaluation kernel (same eval_loop as net_eval_kernel).
template <class Spec>
__global__ void __launch_bounds__(256)
net_eval_spec_kernel(const NetGeo* net, NetPtr R, Job job) {
  extern __shared__ __align__(16) unsigned char smem[];
  eval_loop(Spec::dev(), job, smem + kDescBytes, SpecEval<Spec>{R});
}

#ifndef CK_SPEC_THREADS
#define CK_SPEC_THREADS 512   // threads per CTA of the specialised kernels
#endif

template <class Spec, class Team>
__global__ void __launch_bounds__(CK_SPEC_THREADS, 1)
net_spec_kernel(NetRefs nets, Job job, int ctas) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned rank, team, tsize;
  team_position<Team>(ctas, rank, team, tsize);
  if ((int)team >= job.n_nets) return;
  const NetPtr R = nets.ptr[team];
  team_loop<Team>(Spec::dev(), R, job, ctas, rank, team, tsize, smem + kDescBytes,
                  Spec::geo().prog[PROG_TRAIN].n_phases, SpecPhases<Spec>{R});
}

// ---------------------------------------------------------------------------
// batched evaluation: every CTA is its own team with a private act arena and
// runs PROG_EVAL on images first+blockIdx.x, first+blockIdx.x+gridDim.x, ...
// Same per-neuron arithmetic as training's forward, so labels are identical.
// RunEval(job, ctx, tm) runs the program's phases for one image (interpreted
// or, in the specialised kernels, unrolled at compile time).
template <class RunEval>
__device__ __forceinline__ void eval_loop(const NetGeo& N, const Job& job, unsigned char* work,
                                          const RunEval& run) {
  TeamCtx tm;
  tm.ph = 0;
  tm.sub = nullptr;
  tm.sub_rank = 0;
  tm.rank = 0;
  tm.size = 1;
  tm.gtid = threadIdx.x;
  tm.gsize = blockDim.x;
  tm.gwarp = threadIdx.x >> 5;
  tm.gwarps = blockDim.x >> 5;
  tm.smem = reinterpret_cast<float*>(work);
  tm.smem_floats = job.eval_floats;
  tm.pre = nullptr;
  Ctx ctx;
  ctx.act = job.eval_scratch + (int64_t)blockIdx.x * N.act_size;
  const LayerDev& O = N.L[N.n_layers - 1];
  for (int64_t t = blockIdx.x; t < job.n; t += gridDim.x) {
    ctx.t = t;
    ctx.img = job.first + t;
    set_input(N, job, ctx, tm);
    run(job, ctx, tm);
    const float* y = ctx.act + O.y_off;
    if (threadIdx.x == 0) {
      // numpy argmax: first maximum; a NaN wins at its first occurrence
      int best = 0;
      float bv = y[0];
      for (int j = 1; j < O.cells && !(bv != bv); ++j) {
        const float v = y[j];
        if (v > bv || v != v) { best = j; bv = v; }
      }
      job.pred[t] = best;
    }
    if (job.outputs)
      for (int j = threadIdx.x; j < O.cells; j += blockDim.x) job.outputs[t * O.cells + j] = y[j];
    __syncthreads();
  }
}

#ifndef CK_SPEC_UNIT   // generic-only kernels live in ck_net.cu
struct InterpEval {
  const NetGeo& N;
  const NetPtr& R;
  __device__ __forceinline__ void operator()(const Job& job, Ctx& ctx, TeamCtx& tm) const {
    const Program& P = N.prog[PROG_EVAL];
    for (int ph = 0; ph < P.n_phases; ++ph) {
      run_phase(N, R, P, ph, job, ctx, tm, nullptr);
      __syncthreads();
    }
  }
};

__global__ void __launch_bounds__(256)
net_eval_kernel(const NetGeo* net, NetPtr R, Job job) {
  extern __shared__ __align__(16) unsigned char smem[];
  NetGeo& N = *reinterpret_cast<NetGeo*>(smem);
  load_desc(&N, net);
  eval_loop(N, job, smem + kDescBytes, InterpEval{N, R});
}
#endif  // CK_SPEC_UNIT

}  // namespace ck

