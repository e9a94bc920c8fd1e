"""Benchmark: encrypted LeNet-1 inference throughput (images/s) on B200.

Workload (BASELINE.json config 2 network, "LeNet-1 CKKS N=2^15"): Conv 1->4
5x5 -> x^2 -> avgpool 2 -> Conv 4->12 5x5 -> x^2 -> avgpool 2 -> Flatten ->
FC 192->10, weights N(0,0.1^2), biases N(0,0.01^2) (seeded); CKKS N=2^15,
scale 2^40, q_0 60 bit + 9 x 40 bit + P 60 bit; inputs U[0,1] synthetic
28x28 images packed by the reference's planner at 20 images per ciphertext
(footprint 813 slots).  One step = one pass of the hot path (drop-level,
conv, square, pool, conv, square, pool, flatten, FC -- every rotation, key
switch, masked product, relinearisation and rescale) over B ciphertexts
(20*B images) per GPU.

* ``value``: server-side evaluation with the input ciphertexts resident in
  HBM (images/s, whole job = sum over ranks, weak scaling).
* ``e2e``: the same through the public API from host images: host pack ->
  H2D -> encode + encrypt -> evaluate -> decrypt + decode -> D2H slots.
* ``roofline``: the dominant kernel (hoisted fused conv MAC, conv2) in
  algorithmic 64-bit modular MACs/s against the measured MAC peak of the
  integer pipe on this GPU (microbenchmark, uh_bench_peaks).
* ``cpu_baseline``: the CPU oracle port (op-level schedule, OpenMP over all
  host cores) on one ciphertext (20 images), rank 0 at N=1.

``--impl reference`` runs only that CPU oracle port (the reference package has
no RNS-CKKS implementation; SEAL is absent) on the same config/metric.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "encrypted images/s (LeNet-1 CKKS N=2^15)"
UNIT = "images/s"


def _params():
    from paper_2402_03060_b200.params import HEParams

    return HEParams(poly_degree=1 << 15, depth=9, scale_bits=40, seed=2)


def _model():
    from paper_2402_03060_b200 import planner

    return planner.lenet1(seed=0)


def _config(B, world):
    return {"workload": "BASELINE config 2 network (UniHENN LeNet-1 / M2 topology), reference packing 20 images/ct",
            "model": "LeNet-1 (M2)", "poly_degree": 32768, "scale_bits": 40,
            "moduli_bits": "60 + 9x40 + P60", "images_per_ciphertext": 20, "ciphertexts_per_gpu_per_step": B,
            "global_batch": B * 20 * world, "parallelism": f"dp{world} (independent ciphertexts, keys per rank)",
            "l2": "working set per step >> 126 MB L2 (keys 1.2 GiB, B ciphertexts + hoisted digits)"}


class Clocks:
    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}", "--format=csv,noheader",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1].split()[0]))
                mx = float(parts[2].split()[0])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


class CpuPort:
    """The CPU oracle port of the path (op-level schedule over the C oracle, OpenMP
    over all host cores), keys generated once; one step = one ciphertext
    (20 images) through the whole LeNet-1 schedule."""

    def __init__(self):
        from oracle.ckks_oracle import OracleBackend
        from oracle.slot_sim import SimBackend
        from paper_2402_03060_b200 import driver, planner

        self.driver, self.planner = driver, planner
        self.params, self.m = _params(), _model()
        params = self.params
        self.plan = planner.footprint(self.m, params)
        rng = np.random.default_rng(7)
        self.samples = list(rng.uniform(0, 1, size=(self.plan.capacity, 1, 28, 28)))
        self.be = OracleBackend(params)
        t0 = time.perf_counter()
        seen = {}

        class Rec(SimBackend):  # records which Galois / relin keys the schedule needs, at which level
            def rotate(self, c, r):
                rr = r % params.num_slots
                if rr:
                    seen[rr] = max(seen.get(rr, -1), c.level)
                return super().rotate(c, r)

            def mul_cipher(self, a, b):
                seen["relin"] = max(seen.get("relin", -1), min(a.level, b.level))
                return super().mul_cipher(a, b)

        driver.run_inference(self.m, self.samples, params, plan=self.plan, backend=Rec(params))
        for r, lev in seen.items():
            self.be.relin_key(lev) if r == "relin" else self.be.galois_key(r, lev)
        self.keygen_s = time.perf_counter() - t0
        self.threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))

    def step(self) -> float:
        t0 = time.perf_counter()
        outs, _, _ = self.driver.run_inference(self.m, self.samples, self.params, plan=self.plan, backend=self.be)
        dt = time.perf_counter() - t0
        self.err = max(float(np.max(np.abs(o - self.planner.reference_infer(self.m, s))))
                       for o, s in zip(outs, self.samples))
        return dt

    def describe(self, dt) -> dict:
        cap = self.plan.capacity
        return {"value": cap / dt, "unit": UNIT, "cores": self.threads, "kind": "port",
                "sample": f"1 ciphertext ({cap} images) through the full LeNet-1 schedule per step, op-level, "
                          f"N=2^15, C oracle with OpenMP on {self.threads} threads; {dt:.1f} s/step "
                          f"(+{self.keygen_s:.1f} s keygen, untimed)",
                "max_abs_err_vs_plaintext": self.err}


def cpu_baseline():
    port = CpuPort()
    return port.describe(port.step())


def run_reference(args, rank, world):
    if rank != 0:
        return
    port = CpuPort()
    for _ in range(args.warmup):
        port.step()
    times = [port.step() for _ in range(args.steps)]
    dt = float(np.mean(times))
    cb = port.describe(dt)
    v = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64 (RNS residues)", "data": "synthetic",
            "config": _config(1, 1), "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference = the CPU oracle port of the RNS-CKKS path (the reference package itself is a "
                    "float64 slot simulator without encryption; SEAL is not available)"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=64, help="ciphertexts (x20 images) per GPU per step")
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2402_03060_b200 import _lib, driver, planner
    from paper_2402_03060_b200.he_backend import GpuBackend
    from paper_2402_03060_b200.schedule import CipherState

    params, m = _params(), _model()
    plan = planner.footprint(m, params)
    cap, B = plan.capacity, args.batch
    rng = np.random.default_rng(1000 + rank)
    images = rng.uniform(0.0, 1.0, size=(B, cap, 1, 28, 28))
    groups = [list(images[b]) for b in range(B)]
    planes = driver.pack_groups(m, groups, plan)  # [1][B][slots] host
    be = GpuBackend(params)
    dev = be.device
    stream = torch.cuda.current_stream(dev)

    # device-resident encrypted inputs for `value`
    ct_in = be.encrypt(be.encode_batch(planes[0]))
    layout = driver._input_layout(m, plan)

    def eval_step():
        state, _, _ = driver._run_layers(m, CipherState([ct_in], layout), be, driver.CostModel(),
                                         params.poly_degree, True)
        return state.cts[0]

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        out_ct = eval_step()
    torch.cuda.synchronize()
    # correctness of what is being timed (first ciphertext's 20 images vs the plaintext forward pass)
    final_state, _, _ = driver._run_layers(m, CipherState([ct_in], layout), be, driver.CostModel(),
                                           params.poly_degree, True)
    dec = np.atleast_2d(be.decrypt(final_state.cts[0]))
    got = driver._extract([dec[0]], final_state.layout, plan.offsets[:cap])
    max_err = max(float(np.max(np.abs(y - planner.reference_infer(m, s)))) for y, s in zip(got, groups[0]))
    argmax_ok = all(int(np.argmax(y)) == int(np.argmax(planner.reference_infer(m, s))) for y, s in zip(got, groups[0]))

    # ---- timed region: value ----
    be.kernel_timer = []
    clocks = Clocks(local)
    barrier()
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        out_ct = eval_step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = _lib.launch_count() - l0
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * B * cap * args.steps / (ms / 1e3)
    timers = be.kernel_timer
    be.kernel_timer = None

    # dominant kernel: hoisted conv MAC (both convs), achieved algorithmic MAC/s
    by_level = {}
    for name, lev, a, b, work in timers:
        d = by_level.setdefault(lev, [0.0, 0, 0])
        d[0] += a.elapsed_time(b)
        d[1] += work
        d[2] += 1
    conv_ms = sum(v[0] for v in by_level.values())
    top = max(by_level.items(), key=lambda kv: kv[1][0]) if by_level else None
    rates = np.zeros(16, dtype=np.float64)
    import ctypes

    _lib.call("uh_bench_peaks", be._ctx, ctypes.c_void_p(rates.ctypes.data))
    roofline = None
    if top:
        lev, (tms, work, cnt) = top
        achieved = work / (tms / 1e3) / 1e12
        peak = rates[1] / 1e12
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "conv2_traffic.json")  # from the committed ncu --set full capture
        if os.path.exists(tpath):
            t = json.load(open(tpath))
            if t.get("batch") == B:
                traffic = t["dram_bytes_per_launch"]
        roofline = {"bound": "imad",
                    "bound_note": "integer-pipe bound: the hoisted key-switch inner products (35% of the algorithmic "
                                  "modMACs) and the 60-bit limbs q_0, P run as IMAD.WIDE.U32 chains; the weight-mask "
                                  "contraction of the 40-bit limbs (the other 65% on 5 of 7 limbs) runs exactly on the "
                                  "tensor cores as byte-split u8 IMMA (tensor pipe ~8% active), so frac is the speed "
                                  "relative to an all-IMAD roofline.  Not HBM-bound (9 GB per launch at ~280 GB/s, "
                                  "see hbm_*)",
                    "kernel": f"LeNet conv2 hoisted MAC, level {lev}: k_hoisted_imma (q_1..q_{lev}: key inner "
                              f"products on IMAD + mask contraction on IMMA) + k_hoisted_bank (q_0, P on IMAD)",
                    "achieved": achieved, "peak": peak, "unit": "T modMAC/s", "frac": achieved / peak,
                    "traffic": traffic, "launch_ms": tms / cnt, "algorithmic_macs_per_launch": work / cnt,
                    "share_of_step": tms / ms, "conv_mac_share_of_step": conv_ms / ms,
                    "peak_source": "measured on this GPU: uh_bench_peaks (register-resident 128-bit MAC loop, "
                                   "4 IMAD.WIDE.U32 per MAC)",
                    "peaks_measured": {"imad_per_s": rates[0], "mac128_per_s": rates[1], "mulmod_per_s": rates[2],
                                       "shoup_per_s": rates[4], "fp64_modmac_per_s": rates[5]},
                    "hbm_peak_gbs": 6540.2,
                    "hbm_achieved_gbs": (traffic / (tms / cnt / 1e3) / 1e9) if traffic else None}

    # ---- e2e through the public API from host images ----
    e2e = None
    if not args.no_e2e:
        # the step's inputs: packed slot planes in pinned host memory (copied to the GPU inside the
        # timed region); the step's result: the decrypted logits (gathered on the GPU, copied back)
        planes_h = torch.from_numpy(np.ascontiguousarray(planes)).pin_memory()
        h2d = planes_h[0].numel() * planes_h.element_size()
        n_logits = int(planner.reference_infer(m, np.zeros((m.channels, m.height, m.width))).size)
        d2h = B * cap * n_logits * 8
        barrier()
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.steps):
            outs, _ = driver.infer_batch(m, planes_h, params, plan, be, fused=True)
        s1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = s0.elapsed_time(s1)
        te = torch.tensor([ems], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ems = float(te.item())
        e2e = {"value": world * B * cap * args.steps / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems / args.steps,
               "path": "driver.infer_batch: pinned host planes -> H2D -> GPU encode+encrypt -> fused eval -> "
                       "GPU decrypt+decode+gather -> D2H logits"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline()

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u64 (RNS residues, 64-bit modular)",
                "data": "synthetic (seeded U[0,1] images, seeded N(0,0.1^2) weights)",
                "config": _config(B, world), "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu,
                "gpu_launches": launches, "clocks": clk,
                "check": {"max_abs_err_vs_plaintext": max_err, "argmax_identical": argmax_ok,
                          "images_checked": cap}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
