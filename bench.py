#!/usr/bin/env python
"""Benchmark: target words/s of batched beam-search decode on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

One "step" is one full decode pass of the configured workload (cfg2: the
4000-sentence UN-test-shaped set, beam 5, length buckets of 64) with every
sentence decoded to completion; per-GPU sentence shards are fixed
(length-bucket LPT, sharding.py), so N GPUs split the same 4000 sentences
(strong scaling) with no collective on the data path.

Legs of the JSON line (rank 0 prints one line):
  value     target words/s, whole job; device time of the decode from CUDA
            events on the library's launching stream, max over ranks; source
            ids already prepared on the host (0.5 MB of ids are copied in the
            call), L2 flushed between timed steps.
  e2e       the same metric through the public API Engine.translate_corpus
            on host text lines ("w<id>" tokens): text -> ids -> H2D -> decode
            -> D2H -> detokenised strings, CUDA-event timed, max over ranks.
  roofline  the tensor-core kernel class with the largest in-situ share of
            the machine: algorithmic FLOP per launch / in-situ launch
            duration, measured in the timed mode itself (24 bucket lanes,
            CUDA-graph replay) by device CTA-lifetime accounting
            (AMUN_PROFILE_CTA_TIME), against the sustained bf16 peak; plus
            the whole-pass tensor FLOP rate and every class's SM-time share.
  cpu_baseline  the CPU oracle port of the reference decoder (oracle/,
            reference algorithm in f64 numpy, sentence thread pool with BLAS
            pinned to 1 thread like engine.py:188-190) on a bounded sample of
            the same workload, rank 0 at N=1 only.
--impl reference runs only that CPU decoder (rank 0), K timed steps of a
bounded sample each, and prints the same JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "target words/sec, beam-5 batched decode at 1/2/4/8 B200 vs CPU reference"
UNIT = "target words/s"


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ----------------------------------------------------------------- clocks

_REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x100: "display_clock_setting"}


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clock and throttle
    reasons every 100 ms while the timed region runs."""

    def __init__(self, device: int):
        self.device = device
        self.samples: list[int] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def loop():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for b, name in _REASONS.items():
                            if bits & b:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    self._stop.wait(0.1)

            self._t = threading.Thread(target=loop, daemon=True)
            self._t.start()
        except Exception as e:  # NVML missing: record why
            self.reasons.add(f"nvml_unavailable:{type(e).__name__}")
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------- CPU baseline

def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


CPU_SAMPLE = 200  # fixed stratified 200-sentence subset


def cpu_sample(sentences, n: int):
    """Fixed stratified sample: every len/n-th sentence in length order."""
    order = sorted(range(len(sentences)), key=lambda i: (len(sentences[i]), i))
    stride = max(1, len(order) // n)
    return [sentences[i] for i in order[stride // 2::stride][:n]]


def run_cpu_reference(wl, sentences, threads: int, n_sent: int):
    """Times the CPU port of the reference decoder (oracle/) on a sample."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import beamnmt_oracle as orc
    from paper_1610_01108_b200.model import ModelConfig, random_model
    from paper_1610_01108_b200 import workload as W

    m = random_model(ModelConfig(W.V_SRC, W.V_TRG, W.D_EMB, W.D_H, W.D_ATT), W.MODEL_SEED)
    net = orc.Net({n: a for n, a in m.tensor_items()})
    sample = cpu_sample(sentences, n_sent)
    opts = orc.Opts(wl.beam, wl.max_len_factor, wl.max_len_offset)

    def once():
        t0 = time.perf_counter()
        res = orc.decode_corpus([net], sample, opts, threads=threads)
        wall = time.perf_counter() - t0
        toks = sum(len(h[0].tokens) - (1 if h[0].finished else 0) for h in res)
        return toks, wall

    return net, sample, once


# ----------------------------------------------------------------- ours

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg4", "cfg5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--max-batch", type=int, default=0, help="override the workload's bucket size")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sentences", type=int, default=0)
    ap.add_argument("--subset", type=int, default=0, help="profiling only: stratified subset of the workload")
    ap.add_argument("--bucket", type=int, default=0,
                    help="profiling only: the N sentences around the median length (one realistic length bucket)")
    args = ap.parse_args()
    rank, world, local = env_rank()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # `python bench.py --gpus N`: launch N ranks (one per GPU) ourselves
        # so n_gpus always equals the number of GPUs that decoded
        import socket
        import subprocess

        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.exit(f"--gpus {args.gpus} requested but only {have} CUDA device(s) are visible")
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))

    from paper_1610_01108_b200 import workload as W

    wl = W.WORKLOADS[args.config]
    if args.max_batch:
        wl = W.Workload(**{**wl.__dict__, "batch": args.max_batch})
    sentences = wl.corpus()
    if args.subset:
        sentences = cpu_sample(sentences, args.subset)
    if args.bucket:
        order = sorted(range(len(sentences)), key=lambda i: (len(sentences[i]), i))
        mid = len(order) // 2
        sentences = [sentences[i] for i in order[max(0, mid - args.bucket // 2):][:args.bucket]]
    cfg = {"workload": f"{wl.name}: {wl.description}", "sentences": wl.sentences, "beam": wl.beam,
           "bucket": wl.batch, "cap": f"{wl.max_len_factor}*J+{wl.max_len_offset}",
           "src_tokens": sum(map(len, sentences)),
           "network": "emb500/hid1024/30k attentional GRU enc-dec, random init seed 1",
           "parallelism": f"sentence-sharded x{world} (length-bucket LPT, no collective)",
           "l2": "flushed (256 MiB device write) before every timed step"}

    if args.impl == "reference":
        if rank != 0:
            return
        threads = os.cpu_count() or 1
        # the 200-sentence stratified subset, decoded in
        # disjoint slices: timed step i takes slice i mod n_slices, so the
        # whole K-step run stays within a few minutes; warm-up steps decode
        # a short slice (BLAS / thread-pool warm-up only)
        n = args.cpu_sentences or CPU_SAMPLE
        n_slices = 4
        net, sample, _ = run_cpu_reference(wl, sentences, threads, n)
        slices = [sample[i::n_slices] for i in range(n_slices)]
        from oracle import beamnmt_oracle as orc

        opts = orc.Opts(wl.beam, wl.max_len_factor, wl.max_len_offset)

        def run_slice(sl):
            t0 = time.perf_counter()
            res = orc.decode_corpus([net], sl, opts, threads=threads)
            return sum(len(h[0].tokens) - (1 if h[0].finished else 0) for h in res), time.perf_counter() - t0

        for _ in range(args.warmup):
            run_slice(slices[0][:threads])
        toks = wall = 0.0
        used = []
        for i in range(args.steps):
            t, w = run_slice(slices[i % n_slices])
            used.append(len(slices[i % n_slices]))
            toks += t
            wall += w
        v = toks / wall
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * wall / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (random-init weights, synthetic source ids)", "config": cfg,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "cpu": cpu_model(),
                             "sample": f"step i decodes slice i mod {n_slices} of a fixed stratified "
                                       f"{len(sample)}-sentence {wl.name} subset ({used} sentences per "
                                       f"timed step, {int(toks)} target tokens in {wall:.1f} s)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)
        return

    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1610_01108_b200 import _lib
    from paper_1610_01108_b200.engine import Engine, EngineConfig
    from paper_1610_01108_b200.model import ModelConfig, Vocabulary, random_model
    from paper_1610_01108_b200.sharding import shard_sentences

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def allreduce(x: float, op: str) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX if op == "max" else torch.distributed.ReduceOp.SUM)
        return float(t.item())

    model = random_model(ModelConfig(W.V_SRC, W.V_TRG, W.D_EMB, W.D_H, W.D_ATT), W.MODEL_SEED)
    shard = shard_sentences([len(s) for s in sentences], world, wl.batch, wl.beam, wl.max_len_factor,
                            wl.max_len_offset)[rank]
    local_sents = [sentences[i] for i in shard]
    dm = _lib.device_model(model, local)

    def decode(profile=0):
        return _lib.decode([dm], local_sents, wl.beam, wl.max_len_factor, wl.max_len_offset, False, 1,
                           max_batch=wl.batch, profile=profile)


    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(max(args.warmup, 0)):
        out = decode()
    barrier()
    torch.cuda.synchronize()
    dev_ms, launches, kms, kcount = 0.0, 0, {}, {}
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.fill_(float(_))
            torch.cuda.synchronize()
            out = decode()  # production path: CUDA-graph replay of the decoder step
            dev_ms += out.device_ms
            launches += out.kernel_launches
    torch.cuda.synchronize()
    barrier()
    toks_local = 0
    for i in range(len(local_sents)):
        h = out.hyps(i)[0]
        toks_local += len(h[0]) - (1 if h[2] else 0)
    # Kernel durations.  In the timed mode (24 bucket lanes replaying CUDA
    # graphs concurrently) events cannot sit between the kernels of a graph,
    # so one more pass in exactly that mode runs with device CTA-lifetime
    # accounting (AMUN_PROFILE_CTA_TIME: every CTA adds globaltimer(exit) -
    # globaltimer(entry) to its kernel class): the in-situ numbers below.  An
    # eager single-lane pass with an event pair around every launch gives the
    # launch counts and the kernels' isolated durations (secondary).
    flush.fill_(0.25)
    torch.cuda.synchronize()
    insitu = decode(profile=_lib.PROFILE_CTA_TIME)
    flush.fill_(0.5)
    torch.cuda.synchronize()
    prof = decode(profile=0xFF)
    kms, kcount = dict(prof.kernel_ms), dict(prof.kernel_count)
    breakdown = {k: round(v, 3) for k, v in prof.kernel_ms.items()}
    ms_step = allreduce(dev_ms / args.steps, "max")
    toks = allreduce(float(toks_local), "sum")
    value = toks / (ms_step / 1000.0)

    # ---- roofline per tensor-core kernel class, headline = the class with
    # the largest in-situ share of the machine (CTA lifetime / (148 SMs x
    # pass time)).  Algorithmic work per launch:
    # FLOP = 2 x rows x (fp32 GEMM shape of the reference op); rows = average
    # hypothesis rows per launch of the pass.  The kernels issue three fp16
    # MMAs per product (3xFP16 split), reported as "issued_frac".  In-situ
    # launch duration = mean CTA lifetime of the class (all CTAs of a launch
    # are co-resident).  Peak: the sustained dense bf16 rate (kernels timed
    # inside a long step; kind::f16 runs at the bf16 rate).
    peaks = {}
    pk = REPO / "MEASURED_PEAKS.json"
    if pk.exists():
        peaks = json.loads(pk.read_text())
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    tc_peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 2250.0))
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count
    de, dh, da, V = W.D_EMB, W.D_H, W.D_ATT, W.V_TRG
    lens = sorted(len(s) for s in local_sents)
    rows_sum = n_launch = 0
    for b in range(0, len(lens), wl.batch):
        chunk = lens[b:b + wl.batch]
        steps_b = max(wl.max_len_factor * L + wl.max_len_offset for L in chunk)
        rows_sum += steps_b * len(chunk) * wl.beam
        n_launch += steps_b
    rows = rows_sum / max(1, n_launch)
    shapes = {  # (K, N) of the fp32 GEMM each class computes per hypothesis row
        "query": [(dh, da)],
        "gru_a": [(de + 2 * dh, 3 * dh), (dh, 2 * dh)],  # x W_{z,r,h} + s U_{z,r}
        "gru_b": [(dh, dh)],                            # (r*s) U_h
        "deep_out": [(de + 3 * dh, de)],
        "logits": [(de, V)],
    }
    if not kcount.get("gru_a", 0):
        # projected-context step (decode.cu proj_ok): the context's products
        # come from the encoder-time HX rows, so the step's GEMMs are
        # s [W_att_s | U_z | U_r] and s' W_o^s -- counted as executed
        shapes.update({"query": [(dh, da + 2 * dh)], "deep_out": [(dh, de)]})
        if kcount.get("query", 0) * 2 < kcount.get("deep_out", 0):
            # query folded forward: the deep-output launch also computes the
            # next step's query + s' U_zr; the query class is one launch per bucket
            shapes["deep_out"] = [(dh, de + da + 2 * dh)]
    pass_ms = insitu.device_ms
    sm_ms = {k: insitu.kernel_ms[k] for k in _lib.KERNEL_CLASSES}
    share = {k: round(v / (n_sm * pass_ms), 4) for k, v in sm_ms.items()}
    classes = {}
    pass_flop = 0.0
    for cls, kn in shapes.items():
        n = kcount.get(cls, 0)
        ctas_tot = insitu.kernel_ctas.get(cls, 0)
        if not n or not ctas_tot:
            continue
        flop = sum(2.0 * rows * k * nn for k, nn in kn)
        pass_flop += flop * n
        wbytes = sum(4.0 * k * nn for k, nn in kn)
        ctas = ctas_tot / n
        dur_ms = sm_ms[cls] / ctas_tot  # mean CTA lifetime in situ
        ach = flop / (dur_ms / 1e3) / 1e12
        iso_ms = kms[cls] / n
        classes[cls] = {"launches": int(n), "ctas_per_launch": round(ctas, 1),
                        "gflop_per_launch": round(flop / 1e9, 3),
                        "insitu_launch_ms": round(dur_ms, 4), "achieved_tflops": round(ach, 1),
                        "frac": round(ach / tc_peak, 4), "issued_frac": round(3 * ach / tc_peak, 4),
                        # issued tensor rate on the SMs the launch holds, vs their share of the peak
                        "issued_frac_of_sms_used": round(3 * ach / tc_peak * n_sm / ctas, 4),
                        "weight_gbs": round(wbytes / (dur_ms / 1e3) / 1e9, 1),
                        "share_of_step": share[cls],
                        "isolated_launch_ms": round(iso_ms, 4),
                        "isolated_achieved_tflops": round(flop / (iso_ms / 1e3) / 1e12, 1)}
    dom = max(classes, key=lambda c: sm_ms[c])
    d = classes[dom]
    traffic = None
    tf = REPO / "profiles" / f"{dom}_traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get("dram_bytes_per_launch")
    roofline = {"kernel": dom, "bound": "tensor", "achieved": d["achieved_tflops"], "peak": tc_peak,
                "unit": "TFLOP/s", "frac": d["frac"], "traffic": traffic,
                "issued_frac": d["issued_frac"], "issued_frac_of_sms_used": d["issued_frac_of_sms_used"],
                "ctas_per_launch": d["ctas_per_launch"], "avg_launch_ms": d["insitu_launch_ms"],
                "gflop_per_launch": d["gflop_per_launch"], "rows_per_launch": round(rows, 1),
                "peak_source": "measured (MEASURED_PEAKS.json bf16_tflops_sustained; kind::f16 runs at the bf16 rate)"
                if pk.exists() else "fallback (nominal dense bf16)",
                "share_of_step": d["share_of_step"],
                "timing": "in situ: the timed mode (24 bucket lanes, CUDA-graph replay) with device CTA-lifetime "
                          "accounting (globaltimer per CTA, summed per kernel class); launch duration = mean CTA "
                          "lifetime; share_of_step = class CTA time / (SMs x pass time)",
                "whole_pass": {"tflop_per_pass": round(pass_flop / 1e12, 2),
                               "achieved_tflops": round(pass_flop / (ms_step / 1e3) / 1e12, 1),
                               "frac": round(pass_flop / (ms_step / 1e3) / 1e12 / tc_peak, 4),
                               "issued_frac": round(3 * pass_flop / (ms_step / 1e3) / 1e12 / tc_peak, 4)},
                "tensor_core_classes": classes,
                "insitu_sm_share": share,
                "insitu_pass_ms": round(pass_ms, 2),
                "hbm_peak_gbs": hbm_peak,
                "isolated_kernel_ms_per_step": breakdown,
                "launches_per_step": {k: int(v) for k, v in prof.kernel_count.items()}}

    # ---- e2e through the public API (host text lines)
    e2e = None
    if not args.no_e2e:
        vocab = Vocabulary.from_tokens([f"w{i}" for i in range(2, W.V_SRC)])
        eng = Engine(EngineConfig(model_paths=("<memory>",), src_vocab_path="<memory>", trg_vocab_path="<memory>",
                                  beam_size=wl.beam, max_len_factor=wl.max_len_factor,
                                  max_len_offset=wl.max_len_offset, devices=(local,), max_batch=wl.batch),
                     [model], vocab, vocab, None, None, None, 0, 0.0)
        lines = W.lines_of(local_sents)
        for _ in range(max(args.warmup, 1)):  # same W warm-up steps as the device leg
            eng.translate_corpus(lines)
        barrier()
        torch.cuda.synchronize()
        e2e_ms = 0.0
        h2d = d2h = 0
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            res = eng.translate_corpus(lines)
            ev1.record()
            ev1.synchronize()
            e2e_ms += ev0.elapsed_time(ev1)
            h2d += eng.last_stats["h2d_bytes"]
            d2h += eng.last_stats["d2h_bytes"]
        barrier()
        e2e_toks = allreduce(float(sum(len(r.text.split()) for r in res)), "sum")
        e2e_ms_step = allreduce(e2e_ms / args.steps, "max")
        e2e = {"value": e2e_toks / (e2e_ms_step / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": int(allreduce(h2d / args.steps, "sum")),
               "d2h_bytes_per_step": int(allreduce(d2h / args.steps, "sum")),
               "ms_per_step": e2e_ms_step, "api": "Engine.translate_corpus(lines)"}

    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        n = args.cpu_sentences or CPU_SAMPLE
        _, sample, once = run_cpu_reference(wl, sentences, threads, n)
        t, w = once()
        cpu = {"value": t / w, "unit": UNIT, "cores": threads, "kind": "port", "cpu": cpu_model(),
               "sample": f"{len(sample)} stratified {wl.name} sentences ({sum(map(len, sample))} source, "
                         f"{t} target tokens) in {w:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp32 (fp64 beam scores)",
            "data": "synthetic (random-init weights seed 1, synthetic source ids)", "config": cfg,
            "target_tokens": int(toks), "e2e": e2e, "gpu_launches": int(allreduce(float(launches), "sum")),
            "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks.summary(),
            "source_words_per_s": cfg["src_tokens"] / (ms_step / 1000.0),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
