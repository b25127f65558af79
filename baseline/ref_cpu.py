"""Time the REFERENCE itself (convkit: Python + numba + OpenBLAS) on this
host's cores -- the CPU denominator of bench.py.

The reference is installed once, offline, into baseline/_ref
(`pip install --no-index --no-build-isolation --no-deps --target
baseline/_ref <copy of /root/reference/pkg>`), so it travels to
the GPU box with the repo.  Nothing here is on the product path: bench.py
runs this file as a separate process, one per worker count, each with a FRESH
NUMBA_CACHE_DIR (the reference shares one numba cache entry between its
serial and parallel kernel variants, kernels.py:56-57, so a stale cache would
silently remove the multi-worker speed-up).

Timing follows the reference's own bench (bench.py:49-60): a warm pass over
the samples, then the best of `--windows` windows of at least `--seconds`
each.  Train = NetworkState.train_step(x, t, eta); eval = NetworkState.predict.

    python baseline/ref_cpu.py --workers 16 --nets '{"C3": "input 2x48x48; ..."}'
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time
import warnings

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")


def import_reference():
    """convkit from baseline/_ref (else an installed one); None if absent."""
    if "NUMBA_CACHE_DIR" not in os.environ:
        os.environ["NUMBA_CACHE_DIR"] = tempfile.mkdtemp(prefix="ck_numba_")
    if os.path.isdir(os.path.join(REF, "convkit")) and REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        import convkit
        from convkit import kernels  # noqa: F401  (numba import)
    except Exception:
        return None
    return convkit


def glyph_data(convkit, spec, n, seed=1, split="train"):
    """(n, C, H, W) float32 images + labels: channel c drawn with seed + c
    (SURVEY.md §8d), normalised by the reference's from_bytes."""
    import numpy as np
    from convkit.synth import make_glyph_images
    first = spec.layers[0]
    chans, labels = [], None
    for c in range(first.out_maps):
        img, labels = make_glyph_images(n, spec.n_classes, first.out_width, seed + c, split)
        chans.append(img)
    u8 = np.stack(chans, axis=1)
    ds = convkit.from_bytes(u8, labels, spec.n_classes, split, np.float32)
    return ds.images, ds.labels


def best_rate(step, n_samples, seconds, windows):
    """bench.py:49-60 pattern: warm pass, then the best of `windows` windows."""
    for i in range(n_samples):
        step(i)
    best, total = 0.0, 0
    for _ in range(windows):
        done = 0
        t0 = time.perf_counter()
        while True:
            step(done % n_samples)
            done += 1
            el = time.perf_counter() - t0
            if el >= seconds and done >= n_samples:
                break
        total += done
        best = max(best, done / el)
    return best, total


def measure(convkit, name, arch, what, seconds, windows, samples, eta=1e-3, seed=0):
    import numpy as np
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        spec = convkit.parse_architecture(arch)
    net = convkit.NetworkState(spec, seed, dtype=np.float32)
    x, labels = glyph_data(convkit, spec, samples)
    targets = [convkit.targets_for(int(lb), spec.n_classes) for lb in labels]
    out = {}
    if "train" in what:
        rate, done = best_rate(lambda i: net.train_step(x[i], targets[i], eta), samples,
                               seconds, windows)
        out["train"] = {"value": rate, "images": done}
    if "eval" in what:
        rate, done = best_rate(lambda i: net.predict(x[i]), samples, seconds, windows)
        out["eval"] = {"value": rate, "images": done}
    return out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, required=True)
    ap.add_argument("--nets", required=True, help="JSON {name: architecture string}")
    ap.add_argument("--what", default="train,eval")
    ap.add_argument("--seconds", type=float, default=1.5)
    ap.add_argument("--windows", type=int, default=3)
    ap.add_argument("--samples", default="{}", help="JSON {name: warm-pass images}")
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args(argv)
    t0 = time.perf_counter()
    convkit = import_reference()
    if convkit is None:
        print(json.dumps({"unavailable": "convkit (baseline/_ref) not importable"}))
        return
    from convkit import kernels
    kernels.set_workers(args.workers)
    nets = json.loads(args.nets)
    samples = json.loads(args.samples)
    res = {"workers": kernels.get_workers(), "numba_cache": os.environ["NUMBA_CACHE_DIR"],
           "nets": {}}
    for name, arch in nets.items():
        res["nets"][name] = measure(convkit, name, arch, args.what.split(","), args.seconds,
                                    args.windows, int(samples.get(name, 8)), seed=args.seed)
    res["wall_s"] = time.perf_counter() - t0
    print(json.dumps(res))


if __name__ == "__main__":
    main()
