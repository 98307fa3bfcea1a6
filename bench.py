#!/usr/bin/env python
"""bench.py -- PBS/s of batched 4-bit N=2048 TFHE PBS on B200 (BASELINE.json metric).

A step = one pass of the whole hot path (keyswitch + blind rotation with
modulus switch, ACC init and sample extraction = SURVEY.md §8(a) a1-a5) over
one batch of BASELINE configs[1] (default 131,072 ciphertexts, 8 seeded random
LUTs, set-A parameters, P = 3 exact FFT limbs). Inputs are resident in HBM when
the timed region starts and are larger than L2 (2.1 GB), so no flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl reference]

Multi-GPU (torchrun): weak scaling, each rank bootstraps its own batch with
replicated keys; no data-path collective. The timed region is bracketed by a
barrier + synchronize; time is the max over ranks.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PBS/sec (4-bit, N=2048) on 1 B200; % of FP64/HBM PBS roofline"
UNIT = "PBS/s"
PEAK_FILE = os.path.join(ROOT, "profiles", "r02_fp64_peak.json")      # tools/fp64_peak.py (with its clock log)
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_br_traffic.json")   # tools/ncu_traffic.py


def fp64_peak() -> dict:
    """The FP64 roofline denominator: the measured DFMA burst peak of
    tools/microbench/fp64_peak.cu (best of 10 launches per shape, six shapes;
    sustained 4 s run and the nvidia-smi clock log in the same file)."""
    with open(PEAK_FILE) as f:
        pk = json.load(f)
    return {"tflops": float(pk["burst_tflops"]), "sustained_tflops": float(pk["sustained_tflops"]),
            "clock_derived_tflops": float(pk["clock_derived_tflops"]),
            "sm_mhz": pk.get("sm_mhz_median_under_load"), "source": os.path.relpath(PEAK_FILE, ROOT)}


def br_traffic(batch: int, config: int):
    """dram__bytes_read.sum + dram__bytes_write.sum of the bench's own BR launch
    from the committed ncu capture of the same command (None if it was captured
    for another batch / config)."""
    try:
        with open(TRAFFIC_FILE) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return None, None
    if t.get("batch") != batch or t.get("config") != config:
        return None, None
    return float(t["dram_read_bytes"]) + float(t["dram_write_bytes"]), t


def pbs_flops(P) -> float:
    """Algorithmic FLOPs of one PBS: per CMux, (k+1)l forward and
    (k+1)P inverse M-point FFTs at 5 M log2 M + 6 M (twist), plus (k+1)l(k+1)P M
    complex MACs at 8 flops; times n."""
    M = P.N // 2
    lg = int(np.log2(M))
    fft = 5 * M * lg + 6 * M
    rows, outs = (P.k + 1) * P.pbs_level, (P.k + 1) * P.fft_limbs
    return float(P.n * ((rows + outs) * fft + rows * outs * M * 8))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_baseline(P, sample: int, seed: int) -> dict:
    """The oracle as it stands, on the host's cores, over a bounded sample of the
    same workload (first `sample` ciphertexts of the batch)."""
    import oracle
    from synth import key_randomness, lut_ids, lut_tables, lwe_randomness, messages
    rnd = key_randomness(P, seed)
    ok = oracle.keygen(P, rnd)
    tabs = lut_tables(8, P.p, seed)
    vs = np.stack([oracle.test_polynomial(oracle.encode(tabs[l], P.p), P.p, P.N) for l in range(8)])
    ids = lut_ids(sample, 8, seed)
    m = messages(sample, P.p, seed)
    r = lwe_randomness(P, sample, seed)
    ct = oracle.lwe_encrypt(oracle.encode(m, P.p), ok["big_key"], r["mask"], r["noise"])
    t0 = time.perf_counter()
    out = oracle.pbs(ct, ids, vs, ok["bsk"], ok["ksk"], P)
    dt = time.perf_counter() - t0
    ok_dec = bool(np.array_equal(oracle.lwe_decrypt(out, ok["big_key"], P.p), tabs[ids, m]))
    return {"value": sample / dt, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{sample} PBS of the configs[1] workload (set A, 8 LUTs), exact schoolbook KS+BR+SE, "
                      f"{dt:.1f} s wall, decrypt ok={ok_dec}",
            "seconds": dt}


def run_reference(args):
    """--impl reference: the oracle (the deliberately slow CPU program) as the
    reference arm, rank 0 only."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from synth import get_params
    P = get_params("A")
    steps, warmup = args.steps, args.warmup
    sample = args.ref_sample
    cb = None
    times = []
    for it in range(warmup + steps):
        cb = cpu_baseline(P, sample, args.seed)
        if it >= warmup:
            times.append(cb["seconds"])
    value = sample * steps / sum(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": 1e3 * sum(times) / steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "config": {"workload": f"configs[1] sample of {sample} ciphertexts per step",
                                             "params": "A", "batch": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cb["cores"], "kind": "oracle",
                             "sample": cb["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=131072)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--limbs", type=int, default=3)
    ap.add_argument("--cpu-sample", type=int, default=128)  # ~12 s of oracle work on the 16-core B200 host
    ap.add_argument("--ref-sample", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--config", type=int, default=1, choices=[0, 1],
                    help="BASELINE configs[0] (256 ciphertexts, LUT (3x+1) mod 16) or configs[1] (default)")
    args = ap.parse_args()
    if args.config == 0 and args.batch == 131072:
        args.batch = 256

    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2504_17785_b200 import dist as sdist, silenzio, workload as wl
    from synth import get_params, key_randomness, lut_ids, lut_tables, lwe_randomness, messages

    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    silenzio.load()

    P = get_params("A", fft_limbs=args.limbs, limb_bits={1: 22, 2: 43, 3: 22}[args.limbs])
    B = args.batch
    # ---- setup (not timed): keys replicated per rank, inputs per rank
    rnd = key_randomness(P, args.seed)
    keys = wl.device_keys(P, rnd, dev)
    del rnd
    from synth import config0_table
    tabs = config0_table(P.p) if args.config == 0 else lut_tables(8, P.p, args.seed)
    luts = wl.luts_from_tables(tabs, P.p, P.N, dev)
    in_seed = sdist.input_seed(args.seed, rank)
    ids_np = np.zeros(B, dtype=np.int64) if args.config == 0 else lut_ids(B, 8, in_seed)
    msgs = messages(B, P.p, in_seed)
    r = lwe_randomness(P, B, in_seed)
    ct = wl.encrypt(P, msgs, r, keys["big_key"], dev)
    del r
    ids = torch.from_numpy(ids_np.astype(np.int32)).to(dev)
    small = torch.empty((B, P.n + 1), dtype=torch.int64, device=dev)
    out = torch.empty((B, P.big_dim + 1), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()
    # keyswitch workspace: the KSK byte planes of the tensor-core keyswitch (re-derived every step)
    ks_ws = torch.empty(max(silenzio.keyswitch_workspace_bytes(P, B), 16), dtype=torch.uint8, device=dev)

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        silenzio.keyswitch_batch(ct, keys["ksk"], P, out=small, stream=stream, workspace=ks_ws)
        if ev is not None:
            ev[1].record(stream)
        silenzio.blind_rotate_batch(small, ids, luts, keys["fbsk"], P, out=out, stream=stream)
        if ev is not None:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # correctness of the warm-up output: every ciphertext decrypts to its LUT value
    phase = silenzio.lwe_phase_batch(out, keys["big_key"])
    dec = wl.decode(wl.to_host_u64(phase), P.p)
    failures = int((dec != tabs[ids_np, msgs]).sum())

    clocks = ClockSampler(local)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    # inputs smaller than L2 (configs[0]): flush L2 before every timed step by
    # writing a 256 MB buffer, and time the steps alone (sum of per-step events)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if B * (P.big_dim + 1) * 8 < (256 << 20) else None
    t_start.record(stream)
    for k in range(args.steps):
        if flush is not None:
            flush.zero_()
        step(evs[k])
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = t_start.elapsed_time(t_end)
    if flush is not None:
        total_ms = sum(e[0].elapsed_time(e[2]) for e in evs)
    ks_ms = [e[0].elapsed_time(e[1]) for e in evs]
    br_ms = [e[1].elapsed_time(e[2]) for e in evs]
    total_ms = sdist.max_over_ranks(total_ms, dev)
    failures = sdist.sum_over_ranks(failures, dev)
    ms_per_step = total_ms / args.steps
    value = sdist.aggregate_throughput(world, B, args.steps, total_ms / 1e3)

    # ---- end-to-end through the public host-buffer entry point
    e2e = None
    if not args.no_e2e:
        ct_h = torch.empty((B, P.big_dim + 1), dtype=torch.int64, pin_memory=True)
        ct_h.copy_(ct)
        ids_h = ids.cpu().pin_memory()
        out_h = torch.empty((B, P.big_dim + 1), dtype=torch.int64, pin_memory=True)
        chunk = 16384
        ws = torch.empty(silenzio.pbs_host_workspace_bytes(P, chunk), dtype=torch.uint8, device=dev)
        silenzio.pbs_batch_host(ct_h, ids_h, luts, keys["fbsk"], keys["ksk"], P, out_h, ws, chunk=chunk)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            silenzio.pbs_batch_host(ct_h, ids_h, luts, keys["fbsk"], keys["ksk"], P, out_h, ws, chunk=chunk)
        e2e_s = time.perf_counter() - t0
        e2e_s = sdist.max_over_ranks(e2e_s, dev)
        e2e_ok = bool(torch.equal(out_h, out.cpu()))
        e2e = {"value": sdist.aggregate_throughput(world, B, args.steps, e2e_s), "unit": UNIT,
               "h2d_bytes_per_step": int(B * (P.big_dim + 1) * 8 + B * 4),
               "d2h_bytes_per_step": int(B * (P.big_dim + 1) * 8),
               "api": "silenzio_pbs_batch_host (pinned host buffers, 16384-ciphertext chunks, copies overlapped)",
               "matches_device_path": e2e_ok}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    flops = pbs_flops(P)
    pk = fp64_peak()
    fp64_tf = pk["tflops"]
    traffic, traffic_rec = br_traffic(B, args.config)
    ks_ops = 2.0 * P.big_dim * P.ks_level * (P.n + 1) * 8  # 8 byte-plane int8 GEMM MACs per ciphertext
    launches = int(args.steps * silenzio.pbs_launch_count(P, B))
    br_avg_s = float(np.mean(br_ms)) / 1e3
    achieved = flops * B / br_avg_s / 1e12
    roofline = {"bound": "alu", "pipe": "fp64", "achieved": achieved, "peak": fp64_tf,
                "unit": "TFLOP/s", "frac": achieved / fp64_tf,
                # dram__bytes_read.sum + dram__bytes_write.sum of the bench's own BR launch (ncu, committed capture
                # of the same command; null when the committed capture is for another batch or config)
                "traffic": traffic,
                "traffic_source": (f"{os.path.relpath(TRAFFIC_FILE, ROOT)}: {traffic_rec.get('command')}"
                                   if traffic_rec else "not captured for this batch/config"),
                "algorithmic_bytes": float(silenzio.fourier_bsk_bytes(P) + B * (P.n + 1) * 8
                                           + B * (P.big_dim + 1) * 8 + 8 * P.N * 8),
                "kernel": "blind_rotate_warp_kernel<3>", "algorithmic_flops_per_pbs": flops,
                "kernel_ms": float(np.mean(br_ms)), "keyswitch_ms": float(np.mean(ks_ms)),
                "peak_source": (f"{pk['source']}: measured DFMA burst (best of 10 launches, six shapes, "
                                f"{pk['sm_mhz']} MHz); sustained {pk['sustained_tflops']:.2f}, "
                                f"clock-derived 148x64x2xf_max = {pk['clock_derived_tflops']:.2f}"),
                "frac_vs_clock_derived_peak": achieved / pk["clock_derived_tflops"],
                "keyswitch": {"kernel": "keyswitch_tc_kernel<5> (tcgen05 kind::i8)",
                              "int8_tensor_tops": ks_ops * B / (float(np.mean(ks_ms)) / 1e3) / 1e12,
                              "peak_int8_tops_nominal": 4500.0,
                              "ops_per_ct": ks_ops},
                "pbs_roofline_pbs_per_s": fp64_tf * 1e12 / flops,
                # the stricter P = 1 denominator beside it (an approximate single-limb
                # FFT would need only these flops, but cannot meet the 2^-32 parity bound, DESIGN R20)
                "frac_vs_p1_flops": (pbs_flops(P.with_(fft_limbs=1)) * B / br_avg_s / 1e12) / fp64_tf,
                "frac_of_pbs_roofline_whole_step": value / world / (fp64_tf * 1e12 / flops)}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64/f64", "data": "synthetic",
            "config": {"workload": (f"BASELINE configs[0]: batch {B} per GPU, LUT (3x+1) mod 16, " if args.config == 0
                                    else f"BASELINE configs[1]: batch {B} per GPU, 8 seeded random LUTs over Z_16, ")
                                   + f"set A (n=742,k=1,N=2048,PBS 2^23x1,KS 2^3x5), P={P.fft_limbs} FFT limbs",
                       "batch": B, "global_batch": B * world, "params": "A", "fft_limbs": P.fft_limbs,
                       "limb_bits": P.limb_bits, "parallelism": f"dp{world} (independent ciphertexts)",
                       "l2": (f"inputs {B * (P.big_dim + 1) * 8 / 1e9:.2f} GB per step > 126 MB L2, no flush needed"
                              if flush is None else
                              f"inputs {B * (P.big_dim + 1) * 8 / 1e6:.1f} MB < L2: a 256 MB buffer is written before "
                              "every timed step; time = sum of the per-step events (flush excluded)"),
                       "decrypt_failures": failures},
            "roofline": roofline, "gpu_launches": launches, "clocks": clk}
    if e2e is not None:
        line["e2e"] = e2e
    if not args.no_cpu_baseline and world == 1:
        cb = cpu_baseline(P, args.cpu_sample, args.seed)
        cb.pop("seconds", None)
        line["cpu_baseline"] = cb
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
