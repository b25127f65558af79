"""Benchmark of the online-BP hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2]
                    [--imgs-per-step 2000] [--impl ours|reference]

One STEP is one online-training pass (a weight update after every image) of
the configuration's net over ``--imgs-per-step`` synthetic images that are
already resident in HBM: ONE launch of the persistent training kernel
(ck_net_train_epoch).  The default workload is BASELINE.json configs[1], the
deep MNIST net (C2).  Rank r of N trains its own independent net (init seed
r: a committee member, training.run_experiment semantics), so per-GPU work is
fixed as N grows ("weak").  L2 is flushed (a 256 MiB write) between timed
steps, outside the timed events.

Also reported on the same JSON line:
  eval        test-set evaluation, 10k images sharded over the N ranks, NCCL
              all-gather of predicted labels + all-reduce of the error count
  e2e         the same training metric through the public API
              (training.train_epoch) from pinned HOST bytes: upload, shuffle,
              launch and the loss read back are all inside the timed region
  roofline    the persistent training kernel: algorithmic FP32 FLOPs per
              launch / its CUDA-event duration, against the FP32 SIMT peak
  cpu_baseline  the CPU oracle port (oracle/) on this box's host cores
  clocks      nvidia-smi samples taken during the timed region

``--impl reference`` times the reference's CPU algorithm (the oracle port,
all host threads) on the same config/metric: rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
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


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--imgs-per-step", type=int, default=2000)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--team", default=None,
                    help="kind,ctas,threads for the training kernel (default: engine auto)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="bounded CPU-baseline sample length")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-committee", action="store_true")
    ap.add_argument("--no-deform", action="store_true")
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


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms."""

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
                 "--format=csv,noheader,nounits", "-lms", "200"],
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


def cpu_oracle_rate(spec, data, seconds: float, threads: int, eta=1e-3):
    """Online training images/s of the CPU oracle port on a bounded sample
    (the oracle is test infrastructure: this leg only CHECKS/compares)."""
    from oracle import oracle as orc
    orc.set_threads(threads)
    net = orc.OracleNet(spec, 0)
    targets = np.eye(spec.n_classes, dtype=np.float64) * 2.0 - 1.0
    imgs, labels = data.images, data.labels
    for i in range(min(4, len(imgs))):                    # warm pass
        net.train_step(imgs[i], targets[labels[i]], eta)
    done, i = 0, 0
    t0 = time.perf_counter()
    while True:
        net.train_step(imgs[i], targets[labels[i]], eta)
        done += 1
        i = (i + 1) % len(imgs)
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return done / el, done, el


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU algorithm (oracle port), rank 0 only


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1102_0183_b200.configs import DESCRIPTION, spec_for
    spec = spec_for(args.config)
    data = make_data(spec, 256, 1, "train")
    threads = cpu_threads()
    from oracle import oracle as orc
    orc.set_threads(threads)
    net = orc.OracleNet(spec, 0)
    targets = np.eye(spec.n_classes, dtype=np.float64) * 2.0 - 1.0
    sample = max(8, min(args.imgs_per_step, 256))
    i = 0

    def step():
        nonlocal i
        for _ in range(sample):
            net.train_step(data.images[i], targets[data.labels[i]], 1e-3)
            i = (i + 1) % len(data)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    rate = sample * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config}: {DESCRIPTION[args.config]}, online SGD, "
                               f"{sample} images per step (bounded CPU sample)",
                   "eta": 1e-3},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{sample * args.steps} online steps of {args.config} "
                                   f"(oracle/ck_oracle.c + numpy walk, OpenMP {threads} "
                                   f"threads, {cpu_model()})"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), file=_OUT, flush=True)


# ---------------------------------------------------------------------------
# our arm


def run_ours(args):
    import torch
    import torch.distributed as dist

    import ctypes as C

    import paper_1102_0183_b200 as ck
    from paper_1102_0183_b200 import _lib, multigpu, training
    from paper_1102_0183_b200.configs import DESCRIPTION, spec_for, work_per_image
    from paper_1102_0183_b200.device import DeviceDataset, pin_dataset, upload_bytes

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # under torchrun (any world size, 1 included) the collectives run for real
    use_dist = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ or "RANK" in os.environ
    if use_dist:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if not use_dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    spec = spec_for(args.config)
    work = work_per_image(spec)
    n_img = args.imgs_per_step
    team = tuple(int(v) for v in args.team.split(",")) if args.team else None
    net = ck.NetworkState(spec, rank, device=local, team=team)
    train = make_data(spec, n_img, 1, "train")
    dd = DeviceDataset(train, local)
    stream = torch.cuda.current_stream(local)
    sh = stream.cuda_stream
    rng = np.random.default_rng([rank, 0, 0x5FFE])
    orders = [torch.from_numpy(rng.permutation(n_img).astype(np.int32)).to(dev)
              for _ in range(4)]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    eta = 1e-3

    # -- device-resident training: warm-up, then K timed steps -------------
    for w in range(args.warmup):
        training.train_sequence_async(net, dd, orders[w % 4], eta, sh)
    barrier()
    launches0 = _lib.kernel_launches()
    clocks = ClockSampler(local)
    clocks.start()
    step_ms = []
    for k in range(args.steps):
        flush.fill_(float(k))                       # evict L2 between steps
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        training.train_sequence_async(net, dd, orders[k % 4], eta, sh)
        e.record(stream)
        e.synchronize()
        step_ms.append(s.elapsed_time(e))
    barrier()
    clk = clocks.stop()
    launches = _lib.kernel_launches() - launches0
    my_total = sum(step_ms)
    total_ms = max_over_ranks(my_total)
    value = world * n_img * args.steps / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps

    # -- sharded test-set evaluation + NCCL gather ------------------------
    test = make_data(spec, TEST_IMAGES, 1, "test")
    tdd = DeviceDataset(test, local)
    per = (TEST_IMAGES + world - 1) // world
    first = min(rank * per, TEST_IMAGES)
    mine = max(0, min(per, TEST_IMAGES - first))
    pred = torch.zeros(per, dtype=torch.int32, device=dev)
    gathered = torch.zeros(per * world, dtype=torch.int32, device=dev)
    labels = tdd.labels
    if use_dist:       # evaluate one committee member everywhere: rank 0's weights
        flat = torch.from_numpy(net.flat_parameters()).to(dev)
        dist.broadcast(flat, 0)
        eval_net = ck.NetworkState(spec, 0, device=local)
        eval_net.set_flat_parameters(flat.cpu().numpy())
    else:
        eval_net = net

    def eval_step(engine="exact"):
        if mine:
            training.eval_range_async(eval_net, tdd, first, mine, pred, stream=sh, engine=engine)
        wrong = (pred[:mine] != labels[first:first + mine]).sum().to(torch.int64).reshape(1)
        if use_dist:
            dist.all_gather_into_tensor(gathered, pred)
            dist.all_reduce(wrong)
        else:
            gathered.copy_(pred)
        return wrong

    for _ in range(max(3, args.warmup)):
        eval_step()
    barrier()
    ev_ms = []
    for k in range(args.steps):
        flush.fill_(float(k))
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        wrong = eval_step()
        e.record(stream)
        e.synchronize()
        ev_ms.append(s.elapsed_time(e))
    barrier()
    ev_total = max_over_ranks(sum(ev_ms))
    eval_rate = TEST_IMAGES * args.steps / (ev_total / 1e3)
    err_pct = 100.0 * int(wrong.item()) / TEST_IMAGES
    exact_labels = gathered.clone()

    # -- the same sharded evaluation on the tensor cores (tcgen05 implicit
    # GEMM, fp16 hi/lo split, within tolerance) ---------------------------
    for _ in range(max(3, args.warmup)):
        eval_step("tc")
    barrier()
    tc_ms = []
    for k in range(args.steps):
        flush.fill_(float(k))
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        wrong_tc = eval_step("tc")
        e.record(stream)
        e.synchronize()
        tc_ms.append(s.elapsed_time(e))
    barrier()
    tc_total = max_over_ranks(sum(tc_ms))
    tc_rate = TEST_IMAGES * args.steps / (tc_total / 1e3)
    agree = float((gathered[:TEST_IMAGES] == exact_labels[:TEST_IMAGES]).float().mean().item())
    peaks = {}
    ppath = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(ppath):
        with open(ppath) as f:
            peaks = json.load(f)
    tc_peak = peaks.get("bf16_tflops", 2250.0)
    tc_achieved = work["forward"] * tc_rate / 1e12
    eval_tc = {"value": tc_rate, "unit": UNIT, "test_images": TEST_IMAGES, "scaling": "strong",
               "error_pct": 100.0 * int(wrong_tc.item()) / TEST_IMAGES,
               "label_agreement_with_exact": agree, "ms_per_pass": tc_total / args.steps,
               "engine": "tcgen05 implicit GEMM, fp16 hi/lo split (3 MMAs), f32 accumulate",
               "roofline": {"bound": "tensor", "achieved": tc_achieved, "peak": tc_peak,
                            "unit": "TFLOP/s", "frac": tc_achieved / tc_peak,
                            "peak_basis": "dense 16-bit tensor peak, MEASURED_PEAKS.json "
                                          "bf16_tflops" if "bf16_tflops" in peaks else
                                          "nominal 2.25 PFLOP/s dense 16-bit",
                            "work": "useful forward FLOPs per image (2 per MAC of the "
                                    "reference's sparse tables)"}}

    # -- end to end through the public API from pinned host bytes ----------
    e2e = None
    if not args.no_e2e:
        host = pin_dataset(make_data(spec, n_img, 2, "train"))
        cfg = ck.TrainConfig(epochs=1, eta0=eta, seed=rank)
        h2d = upload_bytes(host) + 4 * n_img            # + the visit order
        for w in range(args.warmup):
            host._device_cache.clear()
            ck.train_epoch(net, host, cfg, w)
        barrier()
        e2e_ms = []
        for k in range(args.steps):
            host._device_cache.clear()                  # re-upload every step
            flush.fill_(float(k))
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            ck.train_epoch(net, host, cfg, k)           # returns the mean loss (D2H)
            e.record(stream)
            e.synchronize()
            e2e_ms.append(s.elapsed_time(e))
        barrier()
        e2e_total = max_over_ranks(sum(e2e_ms))
        e2e = {"value": world * n_img * args.steps / (e2e_total / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8,
               "api": "paper_1102_0183_b200.train_epoch(net, host Dataset, config, epoch)"}

    # -- committee (BASELINE configs[4]): 8 independent C1 nets over the N
    # ranks, each rank's members trained together in one launch per step ---
    committee = None
    if not args.no_committee:
        c_spec = spec_for("C1")
        members = multigpu.nets_for_rank(8, rank, world)
        c_nets = [ck.NetworkState(c_spec, m, device=local) for m in members]
        c_data = make_data(c_spec, n_img, 1, "train")
        c_dd = DeviceDataset(c_data, local)
        handles = (C.c_void_p * len(c_nets))(*[nt.handle.value for nt in c_nets])

        def committee_step(k):
            _lib.call("ck_committee_train_epoch", handles, len(c_nets), c_dd.images_ptr,
                      c_dd.lut_ptr, c_dd.labels.data_ptr(), orders[k % 4].data_ptr(), n_img,
                      float(eta), None, sh)

        if c_nets:
            for w in range(args.warmup):
                committee_step(w)
        barrier()
        c_ms = []
        for k in range(args.steps):
            flush.fill_(float(k))
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            if c_nets:
                committee_step(k)
            e.record(stream)
            e.synchronize()
            c_ms.append(s.elapsed_time(e))
        barrier()
        c_total = max_over_ranks(sum(c_ms))
        committee = {"value": 8 * n_img * args.steps / (c_total / 1e3), "unit": UNIT,
                     "nets": 8, "nets_per_gpu": len(members), "config": "C1",
                     "kernel": c_nets[0].kernel_info() if c_nets else None,
                     "note": "8 independent C1 nets (seeds 0..7), one launch per rank per "
                             "step; total online-training images/s over all nets"}
        for nt in c_nets:
            nt.close()

    # -- on-line deformation (augment.py): the paper's MNIST
    # distortions drawn and applied on the device for every image of the
    # step, then the online pass over the deformed float32 images ----------
    deform = None
    if not args.no_deform:
        from paper_1102_0183_b200 import augment
        dcfg = augment.DeformationConfig(rotate_max=15.0, scale_max=0.15, elastic_sigma=6.0,
                                         elastic_alpha_max=36.0 / 29.0 * 6.0)
        dbuf = torch.empty((n_img, *dd.in_shape), dtype=torch.float32, device=dev)

        def deform_step(k, train_too):
            augment.deform_epoch(dd, dcfg, rank, k, out=dbuf, stream=sh)
            if train_too:
                _lib.call("ck_net_train_epoch", net.handle, dbuf.data_ptr(), None,
                          dd.labels.data_ptr(), orders[k % 4].data_ptr(), n_img, float(eta),
                          None, None, sh)

        res = {}
        for train_too in (False, True):
            for w in range(args.warmup):
                deform_step(w, train_too)
            barrier()
            d_ms = []
            for k in range(args.steps):
                flush.fill_(float(k))
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                deform_step(k, train_too)
                e.record(stream)
                e.synchronize()
                d_ms.append(s.elapsed_time(e))
            barrier()
            res[train_too] = world * n_img * args.steps / (max_over_ranks(sum(d_ms)) / 1e3)
        deform = {"value": res[False], "unit": UNIT, "train_value": res[True],
                  "config": "rotate 15 deg, scale 15%, elastic sigma 6 alpha 7.45 px "
                            "(PAPER MNIST distortions), params drawn on the device",
                  "note": "value: deformation kernel alone (images/s); train_value: "
                          "deformation + online pass over the deformed images"}

    # -- latency budget of one online step (instrumented run, outside the
    # timed region): online training at batch 1 is bound by the chain of
    # dependent phases and their team barriers, not by FLOPs or bytes ----
    latency = None
    try:
        pw, pb = training.profile_phases(net, train.limit(min(n_img, 500)), eta)
        latency = {"phases_per_image": int(len(pw)),
                   "work_us_per_image": float(pw.sum()) / 1e3,
                   "barrier_us_per_image": float(pb.sum()) / 1e3,
                   "per_phase_us": [round(float(w) / 1e3, 2) for w in pw],
                   "note": "slowest CTA's work per phase + the team barrier after it "
                           "(%globaltimer, instrumented launch); the step time is their sum"}
    except Exception as exc:          # instrumentation is diagnostic only
        latency = {"error": str(exc)[:200]}

    # -- roofline of the persistent training kernel ------------------------
    props = torch.cuda.get_device_properties(local)
    sm_max = clk.get("sm_max_mhz") or 1965.0
    peak = props.multi_processor_count * FP32_LANES_PER_SM * 2 * sm_max * 1e6 / 1e12
    kern_ms = statistics.mean(step_ms)            # one launch per step
    achieved = work["train"] * n_img / (kern_ms / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f).get(args.config)
        if tr and tr.get("imgs_per_launch") == n_img:
            traffic = tr.get("dram_bytes")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads()
        rate, done, el = cpu_oracle_rate(spec, train, args.cpu_seconds, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{done} online steps of {args.config} in {el:.1f} s "
                         f"(oracle/ck_oracle.c + numpy walk, OpenMP, {cpu_model()})"}

    if rank == 0:
        kind, ctas, threads_per = net.team()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {
                "workload": f"{args.config}: {DESCRIPTION[args.config]}, online SGD "
                            f"(update after every image), {n_img} images per step, "
                            f"inputs resident in HBM (uint8 + LUT)",
                "imgs_per_step": n_img, "eta": eta,
                "train_mflop_per_img": work["train"] / 1e6,
                "parallelism": f"committee: {world} independent net(s), one per GPU",
                "l2": "flushed (256 MiB write) between timed steps",
                "team": {"kind": ["auto", "cluster", "grid"][kind], "ctas": ctas,
                         "threads": threads_per},
            },
            "gpu_launches": launches,
            "eval": {"value": eval_rate, "unit": UNIT, "test_images": TEST_IMAGES,
                     "scaling": "strong", "error_pct": err_pct,
                     "ms_per_pass": ev_total / args.steps,
                     "collectives": "nccl all_gather(labels) + all_reduce(errors)"
                     if use_dist else "none (single process)",
                     "eval_mflop_per_img": work["forward"] / 1e6},
            "eval_tc": eval_tc,
            "e2e": e2e,
            "committee": committee,
            "deform": deform,
            "latency": latency,
            "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                         "kernel": f"persistent online-training kernel ({net.kernel_info()})",
                         "peak_basis": f"FP32 SIMT: {props.multi_processor_count} SMs x "
                                       f"{FP32_LANES_PER_SM} lanes x 2 FLOP x {sm_max:.0f} MHz "
                                       "(not in MEASURED_PEAKS.json)"},
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line), file=_OUT, flush=True)
    if use_dist:
        dist.destroy_process_group()


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
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
