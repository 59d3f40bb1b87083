"""Benchmark: constrained beam-search decode (beam = 5) of synthetic ConvFwd
problem configs -- BASELINE.json config 2 (65,536 configs per GPU, default
attn model n_a=256, n_s=512, n_d=2, ConvAsm1x1U, membership + resource-budget
predicates).  Prints ONE JSON line.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--precision f16x3]

* value: whole-job configs/s with tokens already resident in HBM; each step
  is one device-resident ks_beam_search_device call over the GPU's 65,536
  configs, timed with CUDA events on the launching stream; L2 is flushed
  (a 512 MiB write) before every timed step; max over ranks.
* e2e: the same workload through the reference-facing host C-ABI
  (ks_beam_search_batch) with host buffers; H2D of tokens and D2H of beams
  and log-probs are inside the timed region.
* roofline: the gate GEMM (dominant kernel), useful FLOPs per launch
  (reference live-hypothesis counts) / its CUDA-event time,
  against MEASURED_PEAKS.json bf16 dense.
* cpu_baseline: the unmodified reference (oracle/_ref, compiled from its own
  sources) on a bounded sample, all host threads, rank 0 only.
* --impl reference: the reference arm itself (same metric/config/unit).
Multi-GPU: one process per GPU (torchrun), configs sharded by rank, no
collective on the data path ("scaling": "weak").
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "problem-configs/sec, constrained beam decode (beam=5)"
UNIT = "configs/s"
from paper_2404_10162_b200 import workloads as WL  # noqa: E402  (pure Python: maps no engine library)

# BASELINE.json configs: cfg2 is the headline (N=1); the others are reported workloads.
# scaling: "weak" = `configs` per GPU; "strong" = `configs` in total, sharded over the GPUs.
WORKLOADS = {k: dict(v, scaling="strong" if k == "cfg3" else "weak") for k, v in WL.WORKLOADS.items()}
WORKLOADS["cfg4"] = dict(model="train", beam=0, configs=4096, greedy=False, train=True, scaling="strong",
                         label="BASELINE config 4: teacher-forced training step, global batch 4096, "
                               "data-parallel with NCCL all-reduce")
TRAIN_METRIC = "training samples/sec, teacher-forced step (batch 4096)"
TRAIN_UNIT = "samples/s"
TRAIN_LR = 1e-3
W = WORKLOADS["cfg2"]
WNAME = "cfg2"
BEAM = W["beam"]


def metric_name():
    """BASELINE.json's metric for the headline (cfg2/cfg3: beam 5); the other
    decode workloads name their own search."""
    if W["greedy"]:
        return "problem-configs/sec, greedy decode"
    if W["beam"] != 5:
        return f"problem-configs/sec, constrained beam decode (beam={W['beam']})"
    return METRIC


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--precision", default="f16x3", choices=["f16x3", "fp32", "bf16"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--configs", type=int, default=None,
                    help="configs per GPU (weak workloads) or in total (cfg3); default: the workload's")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the fixture parity / agreement block")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def model_path(reference=False):
    """The workload's checkpoint (paper_2404_10162_b200/workloads.py): the tracked
    reference-trained default model, or the cfg5 init_model checkpoint (written
    by our byte-identical init_model, or by the reference's in the reference arm)."""
    if W["model"] == "default":
        return WL.DEFAULT_CKPT
    if W["model"] == "cfg5":
        return WL.cfg5_checkpoint_reference() if reference else WL.cfg5_checkpoint_ours()
    return WL.train_checkpoint(reference)


def shard(args, rank, world):
    """Config range [lo, hi) of this rank: weak = `configs` per GPU (rank-major),
    strong = balanced contiguous shards of `configs` in total."""
    from paper_2404_10162_b200.parallel import shard_bounds, weak_shard

    if W["scaling"] == "strong":
        return shard_bounds(args.configs, rank, world)
    return weak_shard(args.configs, rank)


def total_configs(args, world):
    return args.configs if W["scaling"] == "strong" else args.configs * world


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        # the gate GEMMs run inside a step of tens of ms, back to back under the power
        # cap: the sustained figure is the one for them (burst kept in the line too)
        return p.get("bf16_tflops_sustained", p["bf16_tflops"]), p.get("hbm_gbs"), "measured", p["bf16_tflops"]
    except Exception:
        return 1590.0, 6650.0, "fallback", 1590.0


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the sampler is live (first row in) before the timed region starts, so even a
            # region shorter than the 100 ms period is bracketed by samples
            t0 = time.perf_counter()
            while not self.rows and time.perf_counter() - t0 < 3.0:
                time.sleep(0.005)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            n, t0 = len(self.rows), time.perf_counter()
            while len(self.rows) == n and time.perf_counter() - t0 < 0.3:  # one sample after the region
                time.sleep(0.005)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for n, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def engine_libs_mapped():
    """Our engine libraries mapped into this process (/proc/self/maps)."""
    try:
        with open("/proc/self/maps") as f:
            maps = f.read()
    except OSError:
        return []
    names = ("libks_b200", "libkernelseer_b200", "_kernelseer_b200")
    return sorted({l.split()[-1] for l in maps.splitlines() if any(n in l for n in names)})


def assert_no_engine_mapped():
    """The reference arm times the unmodified reference only: none of our
    libraries may be mapped next to it."""
    libs = engine_libs_mapped()
    if libs:
        raise RuntimeError(f"reference arm has engine libraries mapped: {libs}")


def reference_rate(r, tok, desc, path, threads, seconds_target=15.0, max_configs=None):
    """Times the reference's own (constrained) beam search / greedy decode
    (oracle/_ref, parallel_stripes over `threads`) on a prefix of tok sized to
    ~seconds_target; returns (configs/s, configs, seconds)."""
    def run(n):
        t0 = time.perf_counter()
        if W["greedy"]:
            r.greedy(tok[:n], threads)
        else:
            r.beam(tok[:n], BEAM, desc[:n], WL.reference_predicate_text(path), threads)
        return time.perf_counter() - t0

    n0 = min(len(tok), max(threads, 8 if not W["greedy"] else 64))
    rate0 = n0 / run(n0)
    n = int(min(len(tok), max(n0, rate0 * seconds_target)))
    if max_configs:
        n = min(n, max_configs)
    dt = run(n)
    return n / dt, n, dt


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import RefModel

    path = model_path(reference=True)
    r = RefModel(path)
    assert_no_engine_mapped()
    threads = os.cpu_count() or 1
    # the same configs our arm decodes (Rng::derive(2404, i), the reference's own Rng)
    n_pool = min(total_configs(args, args.gpus), 1 << 16)
    desc = r.descriptors(n_pool, WL.SEED)
    tok, bad = r.encode(desc)
    # one step = a bounded sample sized so the whole W+K run ends within minutes
    rate, n, dt = reference_rate(r, tok, desc, path, threads, seconds_target=6.0)
    step_n = max(threads, int(rate * 6.0))
    times = []
    for i in range(args.warmup + args.steps):
        o = (i * step_n) % max(1, len(tok) - step_n)
        r_, n_, dt_ = reference_rate(r, tok[o:], desc[o:], path, threads, seconds_target=6.0, max_configs=step_n)
        if i >= args.warmup:
            times.append((n_, dt_))
    tot_n = sum(t[0] for t in times)
    tot_t = sum(t[1] for t in times)
    value = tot_n / tot_t
    out = {"metric": metric_name(), "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1000.0 * tot_t / args.steps, "higher_is_better": True,
           "scaling": W["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference",
           "config": {"workload": f"{W['label']} (bounded sample per step)", "model": model_label(path),
                      "configs_per_step": int(tot_n / args.steps), "beam": BEAM,
                      "predicates": predicate_label(path),
                      "inputs": "configs 0.. of the workload, Rng::derive(2404, i) over the model vocabulary"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                            "sample": f"{int(tot_n / args.steps)} configs per step, "
                                      f"{'greedy_decode' if W['greedy'] else 'constrained_beam_search'} "
                                      f"via parallel_stripes({threads})"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def model_label(path):
    h = WL.read_header(path)["header"]
    what = {"default": "reference-trained default model (tests/golden/attn_default_trained.ckpt)",
            "cfg5": f"reference init_model(seed 1), heads x{WL.HEAD_SCALE:g}",
            "train": "reference init_model(seed 1), dropout 0.2 / recurrent 0.2"}[W["model"]]
    return (f"{h['variant']} n_a={h['pre_attention_size']} n_s={h['post_attention_size']} "
            f"n_d={h['attention_dense_nodes']}, {h['kernel']}: {what}")


def predicate_label(path):
    if W["greedy"]:
        return "none (greedy)"
    return f"membership + resource_budget(sum values <= {WL.BUDGETS[WL.read_header(path)['header']['kernel']]:g})"


def fixture_check(eng, precision, path, local):
    """Decodes the workload's reference-decoded parity fixture
    (tests/golden/baseline_parity.npz) with the benched
    engine: parity counts under the tie rule (F16X3 / FP32), or decoded-sequence
    agreement with the reference and with F16X3 (BF16, reduced precision)."""
    key = {"cfg1": "cfg1", "cfg2": "cfg2", "cfg3": "cfg2", "cfg5": "cfg5"}.get(WNAME)
    fx_path = os.path.join(ROOT, "tests", "golden", "baseline_parity.npz")
    if key is None or not os.path.exists(fx_path):
        return None
    fx = np.load(fx_path)
    r = {k.split("/", 1)[1]: fx[k] for k in fx.files if k.startswith(key + "/")}
    tie = r["min_gap"] < 1e-4

    def decode(e):
        if W["greedy"]:
            return e.greedy(r["tok"])[:, None, :]
        return e.beam(r["tok"], BEAM, r["desc"], WL.predicate_dicts(path))["tokens"]

    ref_tok = r["tokens"] if r["tokens"].ndim == 3 else r["tokens"][:, None, :]
    g = decode(eng)
    same_full = (g == ref_tok).all(axis=(1, 2))
    same_top1 = (g[:, 0] == ref_tok[:, 0]).all(axis=1)
    out = {"fixture": f"tests/golden/baseline_parity.npz:{key} (reference-decoded)", "configs": int(len(tie)),
           "tie_adjacent": int(tie.sum()), "mismatching_non_tie": int((~same_full & ~tie).sum())}
    if precision == "bf16":
        from paper_2404_10162_b200 import _cabi

        f = decode(_cabi.Engine(path, local, "f16x3"))
        out = {"fixture": out["fixture"], "configs": out["configs"],
               "vs_reference": {"top1": float(same_top1.mean()), "full_list": float(same_full.mean())},
               "vs_f16x3": {"top1": float((g[:, 0] == f[:, 0]).all(axis=1).mean()),
                            "full_list": float((g == f).all(axis=(1, 2)).mean())}}
    return out


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2404_10162_b200 import _cabi

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    path = model_path()
    eng = _cabi.Engine(path, local, args.precision)
    lo, hi = shard(args, rank, world)
    B = hi - lo
    desc = eng.synthetic(B, WL.SEED, lo)  # configs lo..hi-1 of the workload: Rng::derive(2404, i)
    tok = eng.encode(desc)
    preds = [] if W["greedy"] else WL.predicate_dicts(path)
    T = eng.T
    stream = torch.cuda.current_stream()
    d_tok = torch.from_numpy(tok).cuda()
    d_out = {"tokens": torch.empty((B, BEAM, T), dtype=torch.int32, device="cuda"),
             "log_prob": torch.empty((B, BEAM), dtype=torch.float64, device="cuda"),
             "count": torch.empty(B, dtype=torch.int32, device="cuda"),
             "status": torch.empty(B, dtype=torch.int32, device="cuda"),
             "fail_pred": torch.empty(B, dtype=torch.int32, device="cuda"),
             "fail_step": torch.empty(B, dtype=torch.int32, device="cuda")}
    ptrs = {k: v.data_ptr() for k, v in d_out.items()}
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def step():
        eng.beam_device(d_tok.data_ptr(), 0, B, BEAM, preds, ptrs, stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    evs = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.fill_(1)
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            step()
            s1.record(stream)
            evs.append((s0, s1))
        torch.cuda.synchronize()
    launches_per_step = eng.launches()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    value = total_configs(args, world) * args.steps / (ms / 1000.0)

    # roofline of the dominant kernel (lstm_gemm_tc, the gate GEMMs): every launch of one
    # step on the engine stream (CUDA events), algorithmic FLOPs by the reference formula
    # (2 (2n_a + n_s) 4 n_s per decoder hypothesis-step + the encoder's
    # 2 n_a 4 n_a per direction-step) / their summed time; "mma_issued" is what the
    # tensor pipe executed (F16X3: 3 passes; the projected context contracts fewer columns)
    eng.profile_reset(True)
    step()
    torch.cuda.synchronize()
    gemm_ms, gemm_n, useful = eng.profile()
    each_ms, each_fl, each_ex = eng.profile_launches()
    eng.profile_reset(False)
    bf16_peak, hbm_peak, peak_kind, bf16_burst = peaks()
    launch_ms = float(each_ms.mean())
    launch_flops = float(each_fl.mean())
    achieved = float(each_fl.sum()) / (float(each_ms.sum()) / 1000.0) / 1e12
    issued = float(each_ex.sum()) / (float(each_ms.sum()) / 1000.0) / 1e12
    top = each_fl >= each_fl.max() * 0.999
    full_beam = {"launches": int(top.sum()), "ms": float(each_ms[top].mean()),
                 "useful_tflops": float(each_fl[top].mean()) / (float(each_ms[top].mean()) / 1000.0) / 1e12,
                 "mma_issued_tflops": float(each_ex[top].mean()) / (float(each_ms[top].mean()) / 1000.0) / 1e12}
    step_achieved = useful / (gemm_ms / 1000.0) / 1e12 if gemm_ms > 0 else 0.0
    traffic = traffic_of(args.precision, B)

    # end to end through the host C-ABI (host buffers; H2D of tokens and D2H of beams and
    # log-probs inside the timed region)
    host_out = [None]

    def host_call():
        if W["greedy"]:
            eng.greedy(tok)  # ks_greedy_batch: greedy_decode semantics (strict argmax of p)
        else:
            # caller-owned result buffers, reused call after call as a serving loop would
            host_out[0] = eng.beam(tok, BEAM, None, preds, out=host_out[0])

    for _ in range(max(1, args.warmup // 2)):
        host_call()
    if host_out[0] is not None:
        # a serving loop page-locks its long-lived result buffers once (ks_host_register,
        # outside the timed region): the device-to-host copy then lands in them directly
        _cabi.pin_results(host_out[0])
        host_call()
    e2e_t = []
    for _ in range(max(2, args.steps // 2)):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        host_call()
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = sum(e2e_t)
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = total_configs(args, world) * len(e2e_t) / e2e_s
    h2d = B * 7 * 4
    d2h = B * BEAM * T * 4 if W["greedy"] else B * BEAM * T * 4 + B * BEAM * 8 + 4 * B * 4

    parity = None
    if rank == 0 and not args.no_parity:
        try:
            parity = fixture_check(eng, args.precision, path, local)
        except Exception as ex:  # reported, never fatal for the GPU number
            parity = {"error": str(ex)}
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            from oracle.oracle import RefModel, ref_available

            if ref_available():
                threads = os.cpu_count() or 1
                ref_path = model_path(reference=True)
                rate, n, dt = reference_rate(RefModel(ref_path), tok, desc, ref_path, threads, seconds_target=15.0)
                cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                       "sample": f"the first {n} configs of the same workload in {dt:.1f} s (reference "
                                 f"{'greedy_decode' if W['greedy'] else 'constrained_beam_search'}, "
                                 f"parallel_stripes({threads}))"}
        except Exception as ex:
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                   "sample": f"unavailable: {ex}"}
    if rank == 0:
        out = {
            "metric": metric_name(), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": W["scaling"], "vs_baseline": None,
            "dtype": {"f16x3": "f16x3 (fp16 hi/lo split, 3 MMAs, fp32 accumulate; fp32-grade)",
                      "fp32": "fp32", "bf16": "bf16 (fp32 accumulate)"}[args.precision],
            "data": "synthetic",
            "config": {"workload": f"{W['label']}: {total_configs(args, world)} synthetic configs"
                                   f"{' per GPU' if W['scaling'] == 'weak' else ' in total'}",
                       "model": model_label(path),
                       "configs_per_gpu": B, "configs_total": total_configs(args, world), "beam": BEAM,
                       "inputs": "config i = Rng::derive(2404, i) draw over the model vocabulary "
                                 "(ks_synthetic_descriptors; rank r decodes its contiguous shard)",
                       "predicates": predicate_label(path),
                       "l2": "flushed (512 MiB write) before every timed step",
                       "parallelism": f"dp{world} (configs sharded by rank, no collective)"},
            "parity": parity,
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "ks_greedy_batch (host buffers)" if W["greedy"]
                    else "ks_beam_search_batch (host buffers)"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": bf16_peak, "unit": "TFLOP/s",
                         "frac": achieved / bf16_peak, "traffic": traffic["bytes"] if traffic else None,
                         "traffic_source": traffic["source"] if traffic else "no ncu capture for this workload",
                         "kernel": ("lstm_gemm_tc (gate GEMMs + fused LSTM cell, incl. the context projection), "
                                    "all launches of one step" if args.precision != "fp32" else "lstm_step_simt"),
                         "peak_kind": f"{peak_kind} bf16 dense, sustained (MEASURED_PEAKS.json; burst {bf16_burst:g})",
                         "algorithmic": "reference formula (SURVEY 8(d)) FLOPs / summed launch time; the engine "
                                        "skips part of those FLOPs (projected context, position-1 fan-out, parent "
                                        "compaction: DESIGN 5.1-5.1d), so frac can exceed what the tensor pipe "
                                        "issues (mma_issued_frac, 3 MMA passes per F16X3 product)",
                         "useful_flops_per_launch": launch_flops, "launch_ms": launch_ms,
                         "launches_averaged": int(len(each_ms)),
                         "mma_issued_tflops": issued, "mma_issued_frac": issued / bf16_peak,
                         "full_beam_launch": full_beam,
                         "all_gemm_launches": {"per_step": gemm_n, "ms_per_step": gemm_ms,
                                               "useful_tflops": step_achieved,
                                               "share_of_step": gemm_ms / (ms / args.steps)}},
            "cpu_baseline": cpu,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def traffic_of(precision, configs_per_gpu):
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of the full-beam
    gate-GEMM launch from the ncu --set full capture of THIS workload and
    precision (profiles/traffic.json, written by tools/measure_traffic.py), when
    the captured batch matches."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)[WNAME][precision]
    except Exception:
        return None
    if int(t.get("configs_per_gpu", -1)) != int(configs_per_gpu):
        return None
    return {"bytes": t["dram_bytes"], "source": t["source"]}


def train_data(path, B, seed=4):
    """Synthetic teacher-forcing batch: the workload's configs (Rng::derive(2404, i)
    over the model vocabulary, encoded) + uniformly drawn target tokens (numpy,
    seeded: both arms train on identical batches)."""
    from oracle.train_oracle import Checkpoint  # header parsing only
    from paper_2404_10162_b200 import _cabi

    ck = Checkpoint(path)
    h = WL.read_header(path)
    desc = _cabi.synthetic_descriptors(h["inputs"], B, WL.SEED) if not W.get("ref_arm") else None
    if desc is None:
        from oracle.oracle import RefModel
        desc = RefModel(path).descriptors(B, WL.SEED)
    tok = np.stack([np.searchsorted(np.asarray(h["inputs"][f]), desc[:, f]) for f in range(7)], 1).astype(np.int32)
    rng = np.random.default_rng(seed)
    tgt = np.stack([rng.integers(0, v, B) for v in ck.vsizes], 1).astype(np.int32)
    return tok, tgt, ck


def train_flops_per_sample(ck):
    """~3x the forward gate-GEMM FLOPs (forward, dX, dW)."""
    dec = ck.T * 2.0 * (2 * ck.n_a + ck.n_s) * 4 * ck.n_s
    enc = 2 * 7 * 2.0 * ck.n_a * 4 * ck.n_a
    return 3.0 * (dec + enc)


def reference_train_rate(path, tok, tgt, threads, n):
    """The reference's own train_model batch body (oracle/_ref via ref_shim
    ksref_train_step: per-sample tapes over parallel_stripes, / batch, clip,
    Adam) on n samples; returns samples/s."""
    import ctypes as C

    from tests.golden.make_train_fixtures import ref_lib

    L = ref_lib()
    h = L.ksref_load(path.encode())
    trn = L.ksref_trainer_new(TRAIN_LR)
    loss = C.c_double()
    P = lambda a, t: a.ctypes.data_as(C.POINTER(t))
    idx = np.arange(n, dtype=np.int64)
    t0 = time.perf_counter()
    rc = L.ksref_train_step(h, trn, P(np.ascontiguousarray(tok[:n]), C.c_int32),
                            P(np.ascontiguousarray(tgt[:n]), C.c_int32), n, threads, 1, 1, P(idx, C.c_int64),
                            5.0, C.byref(loss))
    dt = time.perf_counter() - t0
    L.ksref_trainer_free(trn)
    L.ksref_free(h)
    if rc:
        raise RuntimeError("reference train step failed")
    return n / dt, dt


def run_train_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    W["ref_arm"] = True  # configs from the reference's own Rng, no engine library
    path = model_path(reference=True)
    tok, tgt, ck = train_data(path, 4096)
    threads = os.cpu_count() or 1
    reference_train_rate(path, tok, tgt, threads, 1)  # loads oracle/_ref
    assert_no_engine_mapped()
    rate0, _ = reference_train_rate(path, tok, tgt, threads, max(threads, 16))
    n = int(min(4096, max(256, rate0 * 6.0)))
    times = []
    for i in range(args.warmup + args.steps):
        r, dt = reference_train_rate(path, tok, tgt, threads, n)
        if i >= args.warmup:
            times.append(dt)
    value = n * len(times) / sum(times)
    out = {"metric": TRAIN_METRIC, "value": value, "unit": TRAIN_UNIT, "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1000.0 * sum(times) / len(times), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": W["label"] + " (bounded sample per step)", "samples_per_step": n,
                      "model": "attn n_a=256 n_s=512 n_d=2, dropout 0.2 / recurrent 0.2 (ModelConfig defaults)"},
           "cpu_baseline": {"value": value, "unit": TRAIN_UNIT, "cores": threads, "kind": "reference",
                            "sample": f"{n} samples per step: train_model batch body (per-sample tapes over "
                                      f"parallel_stripes({threads}), clip, Adam)"},
           "e2e": {"value": value, "unit": TRAIN_UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def run_train(args):
    import torch
    import torch.distributed as dist

    from paper_2404_10162_b200.dptrain import DataParallelTrainer, shard_batch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    path = model_path()
    GB = args.configs  # global batch
    tok, tgt, ck = train_data(path, GB)
    lo, hi = shard_batch(GB, rank, world)
    dp = DataParallelTrainer(path, local, world)
    stream = torch.cuda.current_stream()
    d_tok = torch.from_numpy(tok[lo:hi]).cuda()
    d_tgt = torch.from_numpy(tgt[lo:hi]).cuda()
    d_idx = torch.arange(lo, hi, dtype=torch.int64, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    epoch = [0]

    def step():
        epoch[0] += 1
        dp.step(d_tok, d_tgt, d_idx, GB, epoch[0], 1, TRAIN_LR, 5.0, stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    evs = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            step()
            s1.record(stream)
            evs.append((s0, s1))
        torch.cuda.synchronize()
    launches = dp.tr.launches()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = GB * args.steps / (ms / 1000.0)
    loss, match = dp.stats()

    # end to end: host (pinned) batch -> H2D, step, loss/matches D2H, every step
    h_tok = torch.from_numpy(tok[lo:hi]).pin_memory()
    h_tgt = torch.from_numpy(tgt[lo:hi]).pin_memory()
    e2e_t = []
    for i in range(max(2, args.steps // 2) + 1):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a = h_tok.cuda(non_blocking=True)
        b = h_tgt.cuda(non_blocking=True)
        epoch[0] += 1
        dp.step(a, b, d_idx, GB, epoch[0], 1, TRAIN_LR, 5.0, stream)
        dp.stats()
        if i:
            e2e_t.append(time.perf_counter() - t0)
    e2e_s = sum(e2e_t)
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = GB * len(e2e_t) / e2e_s
    fl = train_flops_per_sample(ck)
    achieved = fl * value / 1e12
    # the trainer's GEMMs run F16X3 (fp16 hi/lo split along a tripled K, one pass of
    # our tcgen05 GEMM, ks_gemm16.cu) -> the measured sustained bf16/fp16 rate;
    # KS_TRAIN_GEMM=fp32 runs every contraction on the fp32 SIMT GEMM
    gemm_mode = os.environ.get("KS_TRAIN_GEMM", "f16x3")
    tf32_peak, _, kind0, _ = peaks()
    tf32_kind = f"{kind0} dense bf16/fp16, sustained (MEASURED_PEAKS.json): F16X3 training GEMMs"
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            from oracle.oracle import ref_available

            if ref_available():
                threads = os.cpu_count() or 1
                r0, _ = reference_train_rate(path, tok, tgt, threads, max(threads, 16))
                n = int(min(GB, max(threads, r0 * 15.0)))
                rate, dt = reference_train_rate(path, tok, tgt, threads, n)
                cpu = {"value": rate, "unit": TRAIN_UNIT, "cores": threads, "kind": "reference",
                       "sample": f"{n} samples in {dt:.1f} s (train_model batch body, parallel_stripes({threads}))"}
        except Exception as ex:
            cpu = {"value": None, "unit": TRAIN_UNIT, "cores": None, "kind": "reference",
                   "sample": f"unavailable: {ex}"}
    if rank == 0:
        out = {"metric": TRAIN_METRIC, "value": value, "unit": TRAIN_UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": ("fp32 (SIMT GEMMs)" if gemm_mode == "fp32" else
                         "fp32-grade (F16X3 tensor-core GEMMs: fp16 hi/lo at per-operand scales, fp32 accumulate; fp32 elsewhere)"), "data": "synthetic",
               "config": {"workload": W["label"], "global_batch": GB, "per_gpu_batch": hi - lo,
                          "model": "attn n_a=256 n_s=512 n_d=2 (random init), dropout 0.2 / recurrent 0.2 "
                                   "(ModelConfig defaults), ConvAsm1x1U T_out=8",
                          "optimizer": f"Adam lr {TRAIN_LR:g}, clip 5.0",
                          "l2": "flushed (512 MiB write) before every timed step",
                          "parallelism": f"dp{world} (batch sharded, NCCL all-reduce of gradients)"},
               "last_loss_per_sample": loss / GB, "last_position_accuracy": match / (GB * ck.T),
               "e2e": {"value": e2e, "unit": TRAIN_UNIT, "h2d_bytes_per_step": int((hi - lo) * (7 + ck.T) * 4),
                       "d2h_bytes_per_step": 16, "api": "DataParallelTrainer.step (ks_trainer_loss_grads + "
                                                        "all-reduce + ks_trainer_apply) from pinned host buffers"},
               "roofline": {"bound": "tensor", "achieved": achieved, "peak": tf32_peak, "unit": "TFLOP/s",
                            "frac": achieved / tf32_peak, "traffic": None,
                            "kernel": f"whole training step: {'fp32 SIMT' if gemm_mode == 'fp32' else 'F16X3 tcgen05 (ks_gemm16.cu)'} GEMMs + fused "
                                      "cell / attention / head / dropout kernels",
                            "peak_kind": tf32_kind,
                            "flops_per_sample": fl, "mma_issued_tflops_upper": 3.0 * achieved},
               "cpu_baseline": cpu, "gpu_launches": launches * args.steps, "clocks": clk.summary()}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    global W, WNAME, BEAM
    args = parse()
    W, WNAME = WORKLOADS[args.workload], args.workload
    BEAM = W["beam"]
    if args.configs is None:
        args.configs = W["configs"]
    if W.get("train"):
        (run_train_reference_arm if args.impl == "reference" else run_train)(args)
    elif args.impl == "reference":
        run_reference_arm(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
