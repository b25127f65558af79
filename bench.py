"""Benchmark of the online-BP hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3]
                    [--imgs-per-step 128] [--impl ours|reference]

One STEP is one online-training pass (a weight update after every image) of
the configuration's net over ``--imgs-per-step`` synthetic glyph images that
are already resident in HBM: ONE launch of the persistent training kernel
(ck_net_train_epoch).  The headline workload is C3, the NORB-shaped net --
the largest BASELINE config by work per image.  Rank r of N
trains its own independent net (init seed r: a committee member,
training.run_experiment semantics), so per-GPU work is fixed as N grows
("weak").  L2 is flushed (a 256 MiB write) between timed steps, outside the
timed events.

On the same JSON line:
  roofline      the training kernel: algorithmic FP32 FLOPs per launch / its
                CUDA-event duration, against the FP32 SIMT peak
  e2e           the same training metric through the public API
                (training.train_epoch) from pinned HOST bytes: upload,
                shuffle, launch and the loss read back inside the timed region
  eval          test-set evaluation (10k images sharded over the N ranks, NCCL
                all-gather of labels + all-reduce of the error count), with
                its own roofline / e2e (training.evaluate from host bytes)
  eval_tc       the same evaluation on the tensor cores (tcgen05 implicit GEMM)
  committee     BASELINE configs[4]: 8 independent C1 nets over the N ranks
  configs       at N=1, the same four-key blocks for C1, C2, C4 and C4'
  cpu_baseline  the REFERENCE itself (convkit + numba from baseline/_ref,
                baseline/ref_cpu.py) on this box's host cores: workers=1 and
                workers=nproc, each in a fresh process with a fresh numba
                cache, and nproc processes x workers=1 in aggregate for
                evaluation and the committee; the oracle port
                (oracle/, OpenMP) is reported beside it
  clocks        nvidia-smi samples taken during the timed regions

``--impl reference`` times the reference's own CPU implementation (convkit
from baseline/_ref, all host cores; the oracle port if convkit is absent) on
the same config, metric and step definition: rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = ("online-train images/sec/GPU and eval images/sec at 1/2/4/8 B200, "
          "% roofline vs CPU")
UNIT = "images/s"
_OUT = sys.stdout   # the JSON line's stream (see _stdout_for_json_only)
FP32_LANES_PER_SM = 128      # B200 SIMT FP32 lanes per SM (2 FLOP per FFMA)
TEST_IMAGES = 10_000
HEADLINE = "C3"
BLOCKS = ("C1", "C2", "C4", "C4F")
# warm-pass images of the CPU reference per config (its bench.py:49-60 pattern)
CPU_SAMPLES = {"C1": 16, "C2": 16, "C3": 4, "C4": 4, "C4F": 2}
ETA = 1e-3


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=HEADLINE)
    ap.add_argument("--imgs-per-step", type=int, default=128)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--blocks", default=",".join(BLOCKS),
                    help="other configs measured at N=1 ('' for none)")
    ap.add_argument("--team", default=None,
                    help="kind,ctas,threads for the training kernel (default: engine auto)")
    ap.add_argument("--cpu-seconds", type=float, default=1.5,
                    help="CPU window length (best of --cpu-windows windows)")
    ap.add_argument("--cpu-windows", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-committee", action="store_true")
    ap.add_argument("--no-deform", action="store_true")
    ap.add_argument("--no-tc", action="store_true")
    ap.add_argument("--tc-train", default="C4F",
                    help="configs also trained on the tensor-core variant (SURVEY 8(f)4)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU/gloo rehearsal of the multi-rank control flow (tests)")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------
# shared helpers


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def make_data(spec, n, seed, split):
    import paper_1102_0183_b200 as ck
    first = spec.layers[0]
    return ck.make_glyph_dataset(n, spec.n_classes, first.out_width, seed=seed, split=split,
                                 channels=first.out_maps)


def config_dict(name, n_img):
    """The `config` object -- identical in both arms (same step definition)."""
    from paper_1102_0183_b200.configs import DESCRIPTION, spec_for, work_per_image
    work = work_per_image(spec_for(name))
    return {"workload": f"{name}: {DESCRIPTION[name]}, online SGD (update after every "
                        f"image), {n_img} synthetic glyph images per step (seed 1)",
            "imgs_per_step": n_img, "eta": ETA,
            "train_mflop_per_img": work["train"] / 1e6,
            "l2": "GPU arm: flushed (256 MiB write) between timed steps; "
                  "inputs resident in HBM (uint8 + LUT)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def load_peaks() -> dict:
    ppath = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(ppath):
        with open(ppath) as f:
            return json.load(f)
    return {}


# ---------------------------------------------------------------------------
# CPU baselines (test infrastructure: the reference and the oracle port are
# only ever timed here, never on the product path)


def _ref_proc_cmd(workers, nets, what, args, samples):
    return [sys.executable, os.path.join(ROOT, "baseline", "ref_cpu.py"),
            "--workers", str(workers), "--nets", json.dumps(nets), "--what", what,
            "--seconds", str(args.cpu_seconds), "--windows", str(args.cpu_windows),
            "--samples", json.dumps(samples)]


def _fresh_env():
    env = dict(os.environ)
    env["NUMBA_CACHE_DIR"] = tempfile.mkdtemp(prefix="ck_numba_")
    env.pop("CUDA_VISIBLE_DEVICES", None)
    return env


def ref_process(workers, nets, what, args, timeout=900):
    """One fresh process running the reference at `workers` workers."""
    samples = {k: CPU_SAMPLES.get(k, 8) for k in nets}
    try:
        out = subprocess.run(_ref_proc_cmd(workers, nets, what, args, samples),
                             capture_output=True, text=True, env=_fresh_env(), timeout=timeout)
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as exc:                # reported, never fatal
        return {"unavailable": f"reference run failed: {str(exc)[:160]}"}


def ref_aggregate(procs, nets, what, args, timeout=900):
    """`procs` concurrent fresh processes x workers=1; summed rates."""
    samples = {k: CPU_SAMPLES.get(k, 8) for k in nets}
    ps = [subprocess.Popen(_ref_proc_cmd(1, nets, what, args, samples), stdout=subprocess.PIPE,
                           stderr=subprocess.DEVNULL, text=True, env=_fresh_env())
          for _ in range(procs)]
    res = []
    for p in ps:
        try:
            out, _ = p.communicate(timeout=timeout)
            res.append(json.loads(out.strip().splitlines()[-1]))
        except Exception:
            p.kill()
    if not res or any("unavailable" in r for r in res):
        return {"unavailable": "aggregate reference run failed"}
    total = {}
    for name in nets:
        total[name] = {w: sum(r["nets"][name][w]["value"] for r in res)
                       for w in res[0]["nets"][name]}
    return {"procs": len(res), "nets": total}


def cpu_port_rate(spec, data, seconds: float, threads: int):
    """Online training images/s of the CPU oracle port (OpenMP) on a
    bounded sample."""
    from oracle import oracle as orc
    orc.set_threads(threads)
    net = orc.OracleNet(spec, 0)
    targets = np.eye(spec.n_classes, dtype=np.float64) * 2.0 - 1.0
    imgs, labels = data.images, data.labels
    for i in range(min(2, len(imgs))):                    # warm pass
        net.train_step(imgs[i], targets[labels[i]], ETA)
    done, i = 0, 0
    t0 = time.perf_counter()
    while True:
        net.train_step(imgs[i], targets[labels[i]], ETA)
        done += 1
        i = (i + 1) % len(imgs)
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return done / el, done, el


def cpu_block(kind, name, w1, wn, agg, nproc, port=None):
    """cpu_baseline object: the best of workers=1, workers=nproc and (when
    measured) the nproc-process aggregate."""
    cands = []
    if w1 is not None:
        cands.append((w1, 1, f"reference workers=1, fresh process"))
    if wn is not None:
        cands.append((wn, nproc, f"reference workers={nproc}, fresh process"))
    if agg is not None:
        cands.append((agg, nproc, f"{nproc} processes x reference workers=1 (aggregate)"))
    if not cands:
        return None
    v, cores, how = max(cands)
    out = {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
           "sample": f"{kind} of {name}: best of {how}; convkit (numba) from baseline/_ref, "
                     f"best of 3 windows after a warm pass (convkit bench.py:49-60), "
                     f"{cpu_model()}",
           "workers_1": w1, "workers_nproc": wn, "aggregate_nproc_x_1": agg, "nproc": nproc}
    if port is not None:
        out["port"] = port
    return out


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation, rank 0 only


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1102_0183_b200.configs import ARCH, spec_for
    spec = spec_for(args.config)
    n_img = args.imgs_per_step
    threads = cpu_threads()
    sys.path.insert(0, os.path.join(ROOT, "baseline"))
    import ref_cpu
    os.environ["NUMBA_CACHE_DIR"] = tempfile.mkdtemp(prefix="ck_numba_")
    convkit = ref_cpu.import_reference()
    orders = [np.random.default_rng([0, k, 0x5FFE]).permutation(n_img) for k in range(4)]
    if convkit is not None:
        from convkit import kernels
        kernels.set_workers(threads)
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rspec = convkit.parse_architecture(ARCH[args.config])
        net = convkit.NetworkState(rspec, 0, dtype=np.float32)
        x, labels = ref_cpu.glyph_data(convkit, rspec, n_img)
        targets = [convkit.targets_for(int(lb), rspec.n_classes) for lb in labels]
        kind = "reference"
        what = (f"convkit NetworkState.train_step (numba kernels, workers={threads}, fresh "
                f"NUMBA_CACHE_DIR) from baseline/_ref")
    else:
        from oracle import oracle as orc
        orc.set_threads(threads)
        net = orc.OracleNet(spec, 0)
        data = make_data(spec, n_img, 1, "train")
        x, labels = data.images, data.labels
        eye = np.eye(spec.n_classes, dtype=np.float64) * 2.0 - 1.0
        targets = [eye[lb] for lb in labels]
        kind = "port"
        what = f"oracle port (oracle/ck_oracle.c + numpy walk, OpenMP {threads} threads)"

    def step(k):
        for i in orders[k % 4]:
            net.train_step(x[i], targets[i], ETA)

    for w in range(args.warmup):
        step(w)
    t0 = time.perf_counter()
    for k in range(args.steps):
        step(k)
    el = time.perf_counter() - t0
    rate = n_img * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(args.config, n_img),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{n_img * args.steps} online steps of {args.config} "
                                   f"({args.steps} steps of {n_img} images after "
                                   f"{args.warmup} warm-up steps): {what}, {cpu_model()}"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), file=_OUT, flush=True)


# ---------------------------------------------------------------------------
# our arm


class Ctx:
    """Per-rank device / process-group plumbing shared by the measurements."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.args = args
        self.rank, self.world, self.local = dist_env()
        if self.world != args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={self.world}")
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        # under torchrun (any world size, 1 included) the collectives run for real
        self.use_dist = (self.world > 1 or "TORCHELASTIC_RUN_ID" in os.environ
                         or "RANK" in os.environ)
        if self.use_dist:
            dist.init_process_group("nccl", device_id=self.dev)
        self.stream = torch.cuda.current_stream(self.local)
        self.sh = self.stream.cuda_stream
        self.flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=self.dev)
        props = torch.cuda.get_device_properties(self.local)
        self.sms = props.multi_processor_count

    def barrier(self):
        if self.use_dist:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, x: float) -> float:
        if not self.use_dist:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def timed(self, fn, steps, warmup):
        """Warm-up, then `steps` calls each bracketed by CUDA events on the
        launching stream (L2 flushed before each, outside the events);
        returns (per-step ms, max-over-ranks total ms)."""
        for w in range(warmup):
            fn(w)
        self.barrier()
        ms = []
        for k in range(steps):
            self.flush.fill_(float(k))
            s = self.torch.cuda.Event(enable_timing=True)
            e = self.torch.cuda.Event(enable_timing=True)
            s.record(self.stream)
            fn(k)
            e.record(self.stream)
            e.synchronize()
            ms.append(s.elapsed_time(e))
        self.barrier()
        return ms, self.max_over_ranks(sum(ms))

    def fp32_peak(self, sm_mhz):
        return self.sms * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12

    def fp32_roofline(self, flops_per_launch, launch_ms, sm_mhz, kernel, traffic=None):
        peak = self.fp32_peak(sm_mhz)
        achieved = flops_per_launch / (launch_ms / 1e3) / 1e12
        return {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": kernel,
                "peak_basis": f"FP32 SIMT: {self.sms} SMs x {FP32_LANES_PER_SM} lanes x 2 FLOP "
                              f"x {sm_mhz:.0f} MHz (MEASURED_PEAKS.json has no FP32 figure)"}


def eval_shard(ctx, n_images):
    """This rank's contiguous test-set shard and the gather buffers
    (multigpu.shard_range: ceil split, the last shards may be short/empty)."""
    from paper_1102_0183_b200.multigpu import shard_range
    torch = ctx.torch
    per = (n_images + ctx.world - 1) // ctx.world
    first, mine = shard_range(n_images, ctx.rank, ctx.world)
    pred = torch.zeros(per, dtype=torch.int32, device=ctx.dev)
    gathered = torch.zeros(per * ctx.world, dtype=torch.int32, device=ctx.dev)
    wrong = torch.zeros(1, dtype=torch.int64, device=ctx.dev)
    return first, mine, pred, gathered, wrong


def sharded_eval_step(ctx, predict_into, labels, first, mine, pred, gathered, wrong):
    """One sharded evaluation: predict this rank's shard into `pred`, count
    its errors, then all-gather the labels and all-reduce the error count."""
    if mine:
        predict_into(first, mine, pred)
    wrong.copy_((pred[:mine] != labels[first:first + mine]).sum().reshape(1))
    if ctx.use_dist:
        ctx.dist.all_gather_into_tensor(gathered, pred)
        ctx.dist.all_reduce(wrong)
    else:
        gathered.copy_(pred)


def latency_floor(name, phases, barrier_us, sm_mhz, fadd_cycles=4):
    """Latency bound of one online step: `phases` dependent team
    barriers at the measured cost, plus every conv layer's reference-order
    forward chain (bias, then n_src * kx * ky dependent f32 FADDs per output
    cell, kernels.py:78-86) at the FADD latency -- work the step cannot
    parallelise or reorder while staying bit-exact.  Everything else (the
    backward sums, FC layers, staging) is counted as free."""
    from paper_1102_0183_b200.configs import spec_for
    spec = spec_for(name)
    chain = 0
    for i, ls in enumerate(spec.layers):
        if ls.kind == "convolutional":
            prev = spec.layers[i - 1]
            fan_in = ls.in_degree if ls.connectivity == "random" else prev.out_maps
            chain += fan_in * ls.kernel[0] * ls.kernel[1]
    chain_us = chain * fadd_cycles / (sm_mhz * 1e6) * 1e6
    return {"us": phases * barrier_us + chain_us, "barriers_us": phases * barrier_us,
            "conv_chain_steps": chain, "conv_chain_us": chain_us,
            "model": f"{phases} barriers x {barrier_us:.2f} us + {chain} dependent FADDs x "
                     f"{fadd_cycles} cycles at {sm_mhz:.0f} MHz"}


def _traffic(name, n_img, kind="train"):
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(tpath):
        return None
    with open(tpath) as f:
        tr = json.load(f).get(f"{name}:{kind}")
    if tr and tr.get("imgs_per_launch") == n_img:
        return tr.get("dram_bytes")
    return None


def measure_config(ctx, name, steps, warmup, sm_mhz, full):
    """Training, evaluation (exact + tensor cores) and their e2e legs for one
    config.  Returns (block dict, net, launches in the timed training)."""
    import paper_1102_0183_b200 as ck
    from paper_1102_0183_b200 import _lib, training
    from paper_1102_0183_b200.configs import spec_for, work_per_image
    from paper_1102_0183_b200.device import DeviceDataset, pin_dataset, upload_bytes
    torch, args = ctx.torch, ctx.args
    spec = spec_for(name)
    work = work_per_image(spec)
    n_img = args.imgs_per_step
    team = tuple(int(v) for v in args.team.split(",")) if args.team else None
    net = ck.NetworkState(spec, ctx.rank, device=ctx.local, team=team)
    train = make_data(spec, n_img, 1, "train")
    dd = DeviceDataset(train, ctx.local)
    rng = np.random.default_rng([ctx.rank, 0, 0x5FFE])
    orders = [torch.from_numpy(rng.permutation(n_img).astype(np.int32)).to(ctx.dev)
              for _ in range(4)]

    # -- device-resident online training -----------------------------------
    launches0 = _lib.kernel_launches()
    step_ms, total = ctx.timed(
        lambda k: training.train_sequence_async(net, dd, orders[k % 4], ETA, ctx.sh),
        steps, warmup)
    # the counter also saw the warm-up steps: scale to the timed ones
    launches = (_lib.kernel_launches() - launches0) * steps // (steps + warmup)
    value = ctx.world * n_img * steps / (total / 1e3)
    block = {"value": value, "unit": UNIT, "ms_per_step": total / steps,
             "imgs_per_step": n_img, "train_mflop_per_img": work["train"] / 1e6,
             "kernel": net.kernel_info(),
             "roofline": ctx.fp32_roofline(work["train"] * n_img, statistics.mean(step_ms),
                                           sm_mhz, f"persistent online-training kernel "
                                                   f"({net.kernel_info()})",
                                           _traffic(name, n_img))}
    block["train_tc"] = None
    if name in args.tc_train.split(",") and not args.no_tc:
        # the opt-in tensor-core training variant (ck_tct.cu): same steps,
        # conv forward / weight gradients / pulls as tcgen05 GEMMs
        plan = net.tct_plan()
        tc_ms, tc_total = ctx.timed(
            lambda k: _lib.call("ck_tct_train_epoch", plan, dd.images_ptr, dd.lut_ptr,
                                dd.labels.data_ptr(), orders[k % 4].data_ptr(), n_img,
                                float(ETA), None, ctx.sh), steps, warmup)
        tc_rate = ctx.world * n_img * steps / (tc_total / 1e3)
        peaks = load_peaks()
        tc_peak = peaks.get("bf16_tflops", 2250.0)
        tc_ach = work["train"] * n_img / (statistics.mean(tc_ms) / 1e3) / 1e12
        block["train_tc"] = {
            "value": tc_rate, "unit": UNIT, "ms_per_step": tc_total / steps,
            "engine": "tcgen05 implicit GEMMs (fp16 hi/lo split, f32 accumulate) for conv "
                      "forward, weight gradients and pulls; one CUDA graph per visit",
            "tolerance": "vs the exact engine: losses 1e-4 rel, weights 2e-4 abs after an "
                         "online run, labels >= 99% (tests/test_gpu_tct.py)",
            "roofline": {"bound": "tensor", "achieved": tc_ach, "peak": tc_peak,
                         "unit": "TFLOP/s", "frac": tc_ach / tc_peak,
                         "work": "algorithmic training FLOPs per image"}}
    block["e2e"] = None
    if not args.no_e2e:
        host = pin_dataset(make_data(spec, n_img, 2, "train"))
        cfg = ck.TrainConfig(epochs=1, eta0=ETA, seed=ctx.rank)

        def e2e_step(k):
            host._device_cache.clear()                  # re-upload every step
            ck.train_epoch(net, host, cfg, k)           # returns the mean loss (D2H)

        _, e2e_total = ctx.timed(e2e_step, steps, warmup)
        block["e2e"] = {"value": ctx.world * n_img * steps / (e2e_total / 1e3), "unit": UNIT,
                        "h2d_bytes_per_step": upload_bytes(host) + 4 * n_img,
                        "d2h_bytes_per_step": 8,
                        "api": "paper_1102_0183_b200.train_epoch(net, host Dataset, config, "
                               "epoch)"}

    # -- sharded test-set evaluation + NCCL gather --------------------------
    test = make_data(spec, TEST_IMAGES, 1, "test")
    tdd = DeviceDataset(test, ctx.local)
    first, mine, pred, gathered, wrong = eval_shard(ctx, TEST_IMAGES)
    if ctx.use_dist:     # evaluate one committee member everywhere: rank 0's weights
        flat = torch.from_numpy(net.flat_parameters()).to(ctx.dev)
        ctx.dist.broadcast(flat, 0)
        eval_net = ck.NetworkState(spec, 0, device=ctx.local)
        eval_net.set_flat_parameters(flat.cpu().numpy())
    else:
        eval_net = net

    def eval_step(engine):
        sharded_eval_step(ctx, lambda f, n, out: training.eval_range_async(
            eval_net, tdd, f, n, out, stream=ctx.sh, engine=engine),
            tdd.labels, first, mine, pred, gathered, wrong)

    ev_steps = steps if full else max(3, min(steps, 5))
    ev_ms, ev_total = ctx.timed(lambda k: eval_step("exact"), ev_steps, max(3, warmup))
    eval_rate = TEST_IMAGES * ev_steps / (ev_total / 1e3)
    exact_labels = gathered.clone()
    ev = {"value": eval_rate, "unit": UNIT, "test_images": TEST_IMAGES, "scaling": "strong",
          "error_pct": 100.0 * int(wrong.item()) / TEST_IMAGES,
          "ms_per_pass": ev_total / ev_steps, "eval_mflop_per_img": work["forward"] / 1e6,
          "collectives": "nccl all_gather(labels) + all_reduce(errors)" if ctx.use_dist
          else "none (single process)",
          "roofline": ctx.fp32_roofline(work["forward"] * mine, statistics.mean(ev_ms), sm_mhz,
                                        "batched exact evaluation kernel (bit-exact "
                                        "reference order, no FMA)",
                                        _traffic(name, TEST_IMAGES, "eval"))}
    ev["e2e"] = None
    if not args.no_e2e:
        from paper_1102_0183_b200 import multigpu
        host_test = pin_dataset(make_data(spec, TEST_IMAGES, 1, "test"))

        def eval_e2e(k):
            host_test._device_cache.clear()
            if ctx.use_dist:                           # shards + NCCL, labels to the host
                multigpu.sharded_evaluate(eval_net, host_test)
            else:
                ck.evaluate(eval_net, host_test)        # labels back to the host

        _, ee_total = ctx.timed(eval_e2e, ev_steps, max(3, warmup))
        ev["e2e"] = {"value": TEST_IMAGES * ev_steps / (ee_total / 1e3), "unit": UNIT,
                     "h2d_bytes_per_step": upload_bytes(host_test),
                     "d2h_bytes_per_step": 4 * TEST_IMAGES,
                     "api": "paper_1102_0183_b200.multigpu.sharded_evaluate(net, host "
                            "Dataset)" if ctx.use_dist else
                            "paper_1102_0183_b200.evaluate(net, host Dataset)"}
    block["eval"] = ev

    # -- the same evaluation on the tensor cores ----------------------------
    block["eval_tc"] = None
    if not args.no_tc:
        tc_ms, tc_total = ctx.timed(lambda k: eval_step("tc"), ev_steps, max(3, warmup))
        tc_rate = TEST_IMAGES * ev_steps / (tc_total / 1e3)
        agree = float((gathered[:TEST_IMAGES] == exact_labels[:TEST_IMAGES]).float()
                      .mean().item())
        peaks = load_peaks()
        tc_peak = peaks.get("bf16_tflops", 2250.0)
        tc_ach = work["forward"] * TEST_IMAGES / ctx.world / (statistics.mean(tc_ms) / 1e3) / 1e12
        block["eval_tc"] = {
            "value": tc_rate, "unit": UNIT, "test_images": TEST_IMAGES, "scaling": "strong",
            "error_pct": 100.0 * int(wrong.item()) / TEST_IMAGES,
            "label_agreement_with_exact": agree, "ms_per_pass": tc_total / ev_steps,
            "engine": "tcgen05 implicit GEMM, fp16 hi/lo split (3 MMAs), f32 accumulate",
            "roofline": {"bound": "tensor", "achieved": tc_ach, "peak": tc_peak,
                         "unit": "TFLOP/s", "frac": tc_ach / tc_peak,
                         "peak_basis": "dense 16-bit tensor peak, MEASURED_PEAKS.json "
                                       "bf16_tflops" if "bf16_tflops" in peaks else
                                       "nominal 2.25 PFLOP/s dense 16-bit",
                         "work": "useful forward FLOPs per image (2 per MAC of the "
                                 "reference's sparse tables)"}}
    if eval_net is not net:
        eval_net.close()
    return block, net, train, launches


def measure_committee(ctx, steps, warmup, sm_mhz):
    """BASELINE configs[4]: 8 independent C1 nets over the N ranks, each
    rank's members trained together in one launch per step."""
    import ctypes as C

    import paper_1102_0183_b200 as ck
    from paper_1102_0183_b200 import _lib, multigpu
    from paper_1102_0183_b200.configs import spec_for, work_per_image
    from paper_1102_0183_b200.device import DeviceDataset, pin_dataset, upload_bytes
    torch = ctx.torch
    n_img = ctx.args.imgs_per_step
    c_spec = spec_for("C1")
    members = multigpu.nets_for_rank(8, ctx.rank, ctx.world)
    c_nets = [ck.NetworkState(c_spec, m, device=ctx.local) for m in members]
    c_dd = DeviceDataset(make_data(c_spec, n_img, 1, "train"), ctx.local)
    rng = np.random.default_rng([0, 0, 0x5FFE])
    orders = [torch.from_numpy(rng.permutation(n_img).astype(np.int32)).to(ctx.dev)
              for _ in range(4)]
    handles = (C.c_void_p * len(c_nets))(*[nt.handle.value for nt in c_nets])

    def committee_step(k):
        if c_nets:
            _lib.call("ck_committee_train_epoch", handles, len(c_nets), c_dd.images_ptr,
                      c_dd.lut_ptr, c_dd.labels.data_ptr(), orders[k % 4].data_ptr(), n_img,
                      float(ETA), None, ctx.sh)

    c_ms, c_total = ctx.timed(committee_step, steps, warmup)
    work = work_per_image(c_spec)["train"]
    out = {"value": 8 * n_img * steps / (c_total / 1e3), "unit": UNIT, "nets": 8,
           "nets_per_gpu": len(members), "config": "C1",
           "kernel": c_nets[0].kernel_info() if c_nets else None,
           "roofline": ctx.fp32_roofline(work * n_img * len(members), statistics.mean(c_ms),
                                         sm_mhz, "persistent training kernel, one team per "
                                                 "net"),
           "note": "8 independent C1 nets (seeds 0..7), one launch per rank per step; "
                   "total online-training images/s over all nets"}
    out["e2e"] = None
    if not ctx.args.no_e2e and c_nets:
        host = pin_dataset(make_data(c_spec, n_img, 2, "train"))
        cfg = ck.TrainConfig(epochs=1, eta0=ETA, seed=0)

        def e2e_step(k):
            host._device_cache.clear()
            ck.train_committee_epoch(c_nets, host, cfg, k)     # mean losses back (D2H)

        _, e_total = ctx.timed(e2e_step, steps, warmup)
        out["e2e"] = {"value": 8 * n_img * steps / (e_total / 1e3), "unit": UNIT,
                      "h2d_bytes_per_step": upload_bytes(host) + 4 * n_img,
                      "d2h_bytes_per_step": 8 * len(c_nets),
                      "api": "paper_1102_0183_b200.train_committee_epoch(nets, host Dataset, "
                             "config, epoch)"}
    for nt in c_nets:
        nt.close()
    return out


def measure_deform(ctx, net, train, steps, warmup):
    """On-line deformation (augment.py): the paper's MNIST
    distortions drawn and applied on the device for every image of the step,
    alone and followed by the online pass over the deformed images."""
    from paper_1102_0183_b200 import _lib, augment
    from paper_1102_0183_b200.device import DeviceDataset
    torch = ctx.torch
    n_img = ctx.args.imgs_per_step
    dd = DeviceDataset(train, ctx.local)
    order = torch.arange(n_img, dtype=torch.int32, device=ctx.dev)
    dcfg = augment.DeformationConfig(rotate_max=15.0, scale_max=0.15, elastic_sigma=6.0,
                                     elastic_alpha_max=36.0 / 29.0 * 6.0)
    dbuf = torch.empty((n_img, *dd.in_shape), dtype=torch.float32, device=ctx.dev)

    def deform_step(k, train_too):
        augment.deform_epoch(dd, dcfg, ctx.rank, k, out=dbuf, stream=ctx.sh)
        if train_too:
            _lib.call("ck_net_train_epoch", net.handle, dbuf.data_ptr(), None,
                      dd.labels.data_ptr(), order.data_ptr(), n_img, float(ETA), None, None,
                      ctx.sh)

    res = {}
    for train_too in (False, True):
        _, tot = ctx.timed(lambda k: deform_step(k, train_too), steps, warmup)
        res[train_too] = ctx.world * n_img * steps / (tot / 1e3)
    return {"value": res[False], "unit": UNIT, "train_value": res[True],
            "config": "rotate 15 deg, scale 15%, elastic sigma 6 alpha 7.45 px "
                      "(PAPER MNIST distortions), params drawn on the device",
            "note": "value: deformation kernel alone (images/s); train_value: "
                    "deformation + online pass over the deformed images"}


def run_ours(args):
    from paper_1102_0183_b200 import training
    ctx = Ctx(args)
    sm_nominal = load_peaks().get("sm_max_mhz", 1965.0)
    clocks = ClockSampler(ctx.local)
    clocks.start()
    head, net, train, launches = measure_config(ctx, args.config, args.steps, args.warmup,
                                                sm_nominal, full=True)
    clk = clocks.stop()
    sm_max = clk.get("sm_max_mhz") or sm_nominal
    if sm_max != sm_nominal:          # restate the FP32 peaks at the box's max clock
        for r in (head["roofline"], head["eval"]["roofline"]):
            fresh = ctx.fp32_roofline(1.0, 1.0, sm_max, r["kernel"])
            r.update(peak=fresh["peak"], frac=r["achieved"] / fresh["peak"],
                     peak_basis=fresh["peak_basis"])
    committee = None if args.no_committee else measure_committee(ctx, args.steps,
                                                                 args.warmup, sm_max)
    deform = None if args.no_deform else measure_deform(ctx, net, train, args.steps,
                                                        args.warmup)

    # latency budget of one online step (instrumented run, outside the timed
    # region): online training at batch 1 is bound by the chain of dependent
    # phases and their team barriers, not by FLOPs or bytes
    try:
        pw, pb = training.profile_phases(net, train.limit(min(args.imgs_per_step, 500)), ETA)
        live = [i for i in range(len(pw)) if pw[i] > 0 or pb[i] > 0]   # (skipped: prepass)
        bar_us = float(pb.sum()) / 1e3
        floor = latency_floor(args.config, len(live), bar_us / max(1, len(live)), sm_nominal)
        step_us = (float(pw.sum()) + float(pb.sum())) / 1e3
        latency = {"phases_per_image": len(live),
                   "work_us_per_image": float(pw.sum()) / 1e3,
                   "barrier_us_per_image": bar_us,
                   "per_phase_us": [round(float(w) / 1e3, 2) for w in pw],
                   "floor": floor, "frac_of_floor": floor["us"] / step_us if step_us else None,
                   "note": "slowest CTA's work per phase + the team barrier after it "
                           "(%globaltimer, instrumented launch); the step time is their sum. "
                           "floor: the latency bound of the online step -- its team "
                           "barriers plus the reference-order conv chains it cannot split"}
    except Exception as exc:          # instrumentation is diagnostic only
        latency = {"error": str(exc)[:200]}
    kind, ctas, threads_per = net.team()
    net.close()

    blocks = {}
    names = [b for b in args.blocks.split(",") if b and b != args.config]
    if ctx.world == 1:
        for name in names:
            blk, bnet, _, _ = measure_config(ctx, name, args.steps, args.warmup, sm_max,
                                             full=False)
            bnet.close()
            blocks[name] = blk

    # -- CPU baselines (rank 0 at N=1; the GPU is idle by now) ---------------
    cpu = {}
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        from paper_1102_0183_b200.configs import ARCH, spec_for
        nproc = cpu_threads()
        nets = {n: ARCH[n] for n in [args.config] + names}
        w1 = ref_process(1, nets, "train,eval", args)
        wn = ref_process(nproc, nets, "train,eval", args)
        agg = ref_aggregate(nproc, {args.config: ARCH[args.config], "C1": ARCH["C1"]},
                            "train,eval", args)
        spec = spec_for(args.config)
        prate, pdone, pel = cpu_port_rate(spec, train, 2.0, nproc)
        port = {"value": prate, "unit": UNIT, "cores": nproc, "kind": "port",
                "sample": f"{pdone} online steps of {args.config} in {pel:.1f} s "
                          f"(oracle/ck_oracle.c + numpy walk, OpenMP {nproc} threads)"}

        def rate(res, name, what):
            try:
                return float(res["nets"][name][what]["value"])
            except (KeyError, TypeError):
                return None

        def agg_rate(name, what):
            try:
                return float(agg["nets"][name][what])
            except (KeyError, TypeError):
                return None

        for name in nets:
            cpu[name] = {
                "train": cpu_block("online training", name, rate(w1, name, "train"),
                                   rate(wn, name, "train"), None, nproc,
                                   port if name == args.config else None),
                "eval": cpu_block("evaluation (predict)", name, rate(w1, name, "eval"),
                                  rate(wn, name, "eval"),
                                  agg_rate(name, "eval") if name == args.config else None,
                                  nproc)}
        cpu["committee"] = cpu_block("committee online training (independent C1 nets)",
                                     "C1", rate(w1, "C1", "train"), None,
                                     agg_rate("C1", "train"), nproc)
        cpu["_raw"] = {"workers_1": w1, "workers_nproc": wn, "aggregate": agg}

    if ctx.rank == 0:
        head_cpu = cpu.get(args.config, {})
        head["eval"]["cpu_baseline"] = head_cpu.get("eval")
        for name, blk in blocks.items():
            blk["cpu_baseline"] = cpu.get(name, {}).get("train")
            blk["eval"]["cpu_baseline"] = cpu.get(name, {}).get("eval")
        if committee is not None:
            committee["cpu_baseline"] = cpu.get("committee")
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": ctx.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": config_dict(args.config, args.imgs_per_step),
            "setup": {"parallelism": f"committee: {ctx.world} independent net(s), one per "
                                     "GPU; evaluation sharded over the GPUs",
                      "team": {"kind": ["auto", "cluster", "grid"][kind], "ctas": ctas,
                               "threads": threads_per},
                      "kernel": head["kernel"]},
            "gpu_launches": launches,
            "roofline": head["roofline"],
            "cpu_baseline": head_cpu.get("train"),
            "e2e": head["e2e"],
            "eval": head["eval"],
            "eval_tc": head["eval_tc"],
            "committee": committee,
            "deform": deform,
            "latency": latency,
            "configs": blocks,
            "cpu_raw": cpu.get("_raw"),
            "clocks": clk,
        }
        print(json.dumps(line), file=_OUT, flush=True)
    if ctx.use_dist:
        ctx.dist.destroy_process_group()


class DryCtx(Ctx):
    """Ctx on CPU over gloo with wall-clock timing: the --dry-run rehearsal
    of the N-rank control flow (rank roles, shards, collectives, max over
    ranks, rank-0 output) without a GPU (tests/test_multigpu_host.py)."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.args = args
        self.rank, self.world, self.local = dist_env()
        if self.world != args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={self.world}")
        self.dev = torch.device("cpu")
        self.use_dist = self.world > 1 or "RANK" in os.environ
        if self.use_dist:
            dist.init_process_group("gloo")
        self.sms = 148

    def barrier(self):
        if self.use_dist:
            self.dist.barrier()

    def timed(self, fn, steps, warmup):
        for w in range(warmup):
            fn(w)
        self.barrier()
        ms = []
        for k in range(steps):
            t0 = time.perf_counter()
            fn(k)
            ms.append(1e3 * (time.perf_counter() - t0))
        self.barrier()
        return ms, self.max_over_ranks(sum(ms))


def run_dry(args):
    """Stand-in work, real multi-rank plumbing: each rank 'trains' its own net
    (weak scaling, rank-dependent duration so max-over-ranks matters), the
    test set is evaluated in shards with a stand-in predictor, gathered and
    reduced, committee members are split with multigpu.nets_for_rank."""
    from paper_1102_0183_b200 import multigpu
    ctx = DryCtx(args)
    torch = ctx.torch
    n_img = args.imgs_per_step
    step_ms, total = ctx.timed(lambda k: time.sleep(0.002 * (1 + ctx.rank)), args.steps,
                               args.warmup)
    labels = torch.as_tensor(np.arange(TEST_IMAGES) % 10, dtype=torch.int32)
    first, mine, pred, gathered, wrong = eval_shard(ctx, TEST_IMAGES)

    def predict_into(f, n, out):
        idx = torch.arange(f, f + n, dtype=torch.int32)
        out[:n] = torch.where(idx % 7 == 3, (idx + 1) % 10, idx % 10)

    sharded_eval_step(ctx, predict_into, labels, first, mine, pred, gathered, wrong)
    weights = torch.full((5,), float(ctx.rank))
    if ctx.use_dist:
        ctx.dist.broadcast(weights, 0)
    members = multigpu.nets_for_rank(8, ctx.rank, ctx.world)
    counts = torch.tensor([len(members)], dtype=torch.int64)
    if ctx.use_dist:
        ctx.dist.all_reduce(counts)
    if ctx.rank == 0:
        line = {"metric": METRIC, "value": ctx.world * n_img * args.steps / (total / 1e3),
                "unit": UNIT, "n_gpus": ctx.world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": total / args.steps, "dry_run": True,
                "my_ms_per_step": sum(step_ms) / args.steps,
                "eval": {"labels": gathered[:TEST_IMAGES].tolist()[:50],
                         "labels_ok": bool((gathered[:TEST_IMAGES] ==
                                            torch.where(torch.arange(TEST_IMAGES) % 7 == 3,
                                                        (torch.arange(TEST_IMAGES) + 1) % 10,
                                                        torch.arange(TEST_IMAGES) % 10)
                                            ).all()),
                         "wrong": int(wrong.item())},
                "broadcast_weights": weights.tolist(), "committee_members": int(counts.item())}
        print(json.dumps(line), file=_OUT, flush=True)
    if ctx.use_dist:
        ctx.dist.destroy_process_group()


def _stdout_for_json_only():
    """Route everything native code prints (NCCL's version banner, ...) to
    stderr; return a writer for the original stdout, which gets the JSON line
    and nothing else."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    return os.fdopen(saved, "w")


def main(argv=None):
    args = parse_args(argv)
    global _OUT
    _OUT = _stdout_for_json_only()
    if args.impl == "reference":
        run_reference(args)
    elif args.dry_run:
        run_dry(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
