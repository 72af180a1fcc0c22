#!/usr/bin/env python
"""bench.py -- fused-gate state-vector update throughput on B200.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` prints ONE
JSON line on rank 0.  A "step" is one whole-circuit simulation through the
C ABI: sv_set_basis(|0..0>) + sv_apply_circuit(all gates of the workload)
(planning included), i.e. one pass of every SURVEY.md 8(a) row.

Workload at N=1: BASELINE.json configs[1] = c2, the 30-qubit 5x6-grid random
circuit (20 cycles, sqrt X/Y/W + fSim(pi/2, pi/6)), complex64 state (8 GiB,
far larger than the 126 MB L2, so no flush is needed between steps).
N > 1 (torchrun, one rank per GPU): the weak-scaling ladder of BASELINE.json
configs[4] (n = 34 + log2 N, 128 GiB per GPU; --config ladder, the default) or
c4 strong scaling (--config c4).

metric/value: BASELINE.json's metric "fused-gate state-vector update GB/s (% of
HBM peak); sec/circuit".  value = the state-update bandwidth the fused passes
achieve over the whole circuit: algorithmic HBM bytes of all passes (2 x 8 B
per amplitude per fused pass) / sec per circuit, summed
over ranks.  pct_of_hbm_peak = value per GPU / the measured HBM copy peak;
sec_per_circuit and gate_equiv_gbs (gates x 16 B x 2^n / sec, the bandwidth a
one-pass-per-gate simulator would need) are reported beside it.  The
`roofline` object is the dominant kernel (the fused gate-group pass: the
tcgen05 tensor-core kernel when it ran, else the CUDA-core FMA kernel).
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused-gate state-vector update GB/s (% of HBM peak); sec/circuit at n=30–37"
UNIT = "GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="", help="c1..c5, ladder (weak, N>1 default) or a ladder n (34..37)")
    ap.add_argument("--dtype", default="c64", choices=["c64", "c128"])
    ap.add_argument("--kmax", type=int, default=0)
    ap.add_argument("--budget", type=int, default=0)
    ap.add_argument("--tile-bits", type=int, default=0)
    ap.add_argument("--low-bits", type=int, default=0)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--virtual-g", type=int, default=0,
                    help="N=1 only: emulate 2^g ranks on the one GPU (virtual shards: every pass per shard, "
                         "remaps through the pack -> exchange -> unpack path)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--oracle-gates", type=int, default=24, help="cpu_baseline sample size (gates)")
    ap.add_argument("--sweep", default="", help="comma list of budgets to sweep (extra output lines to stderr)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
def workload(cfg, world):
    """N=1: c2 by default.  N>1: the weak-scaling ladder n = 34 + log2(N) (BASELINE.json
    configs[4]) unless --config names a config (c4: strong scaling)."""
    from inputs import circuits as C
    if not cfg:
        cfg = "c2" if world == 1 else "ladder"
    if cfg == "ladder":
        return C.weak_ladder(34 + world.bit_length() - 1)
    if cfg.startswith("c"):
        return C.config(int(cfg[1:]))
    return C.weak_ladder(int(cfg))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.rows = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def peaks():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(tc=False):
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of the dominant
    kernel from the committed ncu --set full summary (profiles/)."""
    p = os.path.join(ROOT, "profiles", "tc_pass_traffic.json" if tc else "tile_pass_traffic.json")
    try:
        return json.load(open(p)).get("dram_bytes_per_launch")
    except Exception:
        return None


def tensor_peak():
    """tf32 dense peak: the measured sustained bf16 GEMM rate (MEASURED_PEAKS.json; the
    passes run inside a long step) x the nominal tf32/bf16 ratio 1.1/2.25 (B200_PROFILING.md)."""
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp.get("bf16_tflops_sustained") or mp["bf16_tflops"]) * 1.1 / 2.25, \
            "measured bf16 sustained x nominal tf32/bf16 (1.1/2.25)"
    except Exception:
        return 1400.0 * 1.1 / 2.25, "fallback 1.4 PF bf16 sustained x 1.1/2.25"


def roof(tc, gbs, hbm, peak_kind, tflops, fp32_peak, tile_bytes, launches, tile_ms, flops_per_step, tc_tflops,
         tc_flops_per_step):
    """Roofline of the dominant kernel, the fused gate-group pass.  Tensor-core kernel
    (k_tc_group_pass): bound = HBM (the operator MMAs are far from the tensor peak), with
    the tensor pipe's fraction beside it.  CUDA-core kernel (k_group_pass): HBM or the FP32
    FMA pipe, whichever fraction is higher."""
    if gbs is None:
        return None
    f_hbm = gbs / hbm
    f_alu = tflops / fp32_peak if tflops else 0.0
    tpk, tpk_kind = tensor_peak()
    common = {"kernel": "k_tc_group_pass (tcgen05 3xTF32 gate-group pass)" if tc else
              "k_group_pass (CUDA-core FMA gate-group pass)",
              "bytes_per_launch": tile_bytes, "launches": launches,
              "avg_launch_ms": tile_ms / max(1, launches), "traffic": ncu_traffic(tc),
              "hbm": {"achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": f_hbm, "peak_kind": peak_kind},
              "alu": {"achieved": tflops, "peak": fp32_peak, "unit": "TFLOP/s", "frac": f_alu,
                      "flops_per_step": flops_per_step,
                      "what": "algorithmic complex flops of the fused programs (8 x 2^k per k-qubit matrix)",
                      "peak_kind": "derived: 148 SMs x 128 FP32 lanes x 2 x sm_max_mhz"}}
    if tc:
        common["tensor"] = {"achieved": tc_tflops, "peak": tpk, "unit": "TFLOP/s",
                            "frac": (tc_tflops / tpk) if tc_tflops else 0.0, "flops_per_step": tc_flops_per_step,
                            "what": "tcgen05 kind::tf32 flops issued (3 products per operator step)",
                            "peak_kind": tpk_kind}
        return dict(bound="hbm", achieved=gbs, peak=hbm, unit="GB/s", frac=f_hbm, **common)
    if f_alu > f_hbm:
        return dict(bound="alu", achieved=tflops, peak=fp32_peak, unit="TFLOP/s", frac=f_alu, **common)
    return dict(bound="hbm", achieved=gbs, peak=hbm, unit="GB/s", frac=f_hbm, **common)


# ---------------------------------------------------------------------------
def oracle_fit(circ):
    """(n, gates, x0, note) for timing the complex128 oracle on the host: the workload itself
    when its 16 * 2^n-byte state fits in 40% of the available host RAM, else the same circuit
    restricted to its lowest n' qubits (gates touching higher qubits dropped) -- the metric is
    per amplitude, so the rate is comparable."""
    n = circ.n
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 1 << 62
    m = n
    while m > 10 and (16 << m) > 0.4 * avail:
        m -= 1
    if m == n:
        return n, list(circ.gates), circ.x0, ""
    gates = [g for g in circ.gates if all(q < m for q in g[1])]
    return m, gates, circ.x0 & ((1 << m) - 1), \
        f"; the n={n} complex128 state exceeds host RAM, so the circuit restricted to qubits 0..{m - 1}"


def oracle_sample(circ, ngates, threads):
    """Time the CPU oracle (as it stands) on the first `ngates` gates of circ."""
    import numpy as np
    import oracle
    n, gates, x0, note = oracle_fit(circ)
    psi = np.empty(1 << n, dtype=np.complex128)
    lib = oracle.lib()
    ngates = min(ngates, len(gates))
    arr, keep = oracle._marshal(gates[:ngates])
    t0 = time.perf_counter()
    lib.oracle_run(n, x0, psi.ctypes.data, arr, ngates, threads)
    t = time.perf_counter() - t0
    del psi
    return t, n, ngates, note


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(args, circ):
    """`--impl reference`: the CPU oracle (the deliberately slow, plain
    complex128 program of oracle/) on the host cores, on bounded samples."""
    import numpy as np
    import oracle
    cores = cpu_cores()
    n, ogates, x0, note = oracle_fit(circ)
    gpp = 4                                  # gates per step (bounded sample)
    psi = np.empty(1 << n, dtype=np.complex128)
    lib = oracle.lib()
    psi[:] = 0
    psi[x0] = 1
    G = len(ogates)
    pos = 0

    def step():
        nonlocal pos
        gs = [ogates[(pos + i) % G] for i in range(gpp)]
        pos += gpp
        arr, keep = oracle._marshal(gs)
        lib.oracle_apply(n, psi.ctypes.data, arr, gpp, cores)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    t = time.perf_counter() - t0
    per_gate = t / (args.steps * gpp)
    value = 2 * 16 * (1 << n) / per_gate / 1e9        # state-update GB/s: each gate reads + writes the c128 state
    G = len(circ.gates)
    sec_circ = per_gate * G * 2.0 ** (circ.n - n)      # the whole workload at that per-amplitude rate
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE.json configs[1] circuit)",
            "config": {"workload": circ.name, "n": circ.n, "gates": G, "state": "complex128 (oracle)",
                       "step": f"{gpp} gates of the circuit, gate by gate (one full read + write of the state per gate)",
                       "l2": "state >> L2"},
            "sec_per_circuit": sec_circ,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} steps x {gpp} gates of {circ.name} (n={n}), complex128, "
                                       f"{cores} OpenMP threads; sec/circuit extrapolated x{G}/gate{note}"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    circ = workload(args.config, world)
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, circ)
        return

    import numpy as np
    import torch
    import paper_2008_00216_b200 as stv

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as td
        td.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        uid = [stv.nccl_unique_id() if rank == 0 else None]
        td.broadcast_object_list(uid, src=0)
        dist = {"rank": rank, "world": world, "uid": uid[0]}
    stv.lib()
    n = circ.n
    st = stv.State(n, args.dtype, dist=dist, virtual_g=args.virtual_g if world == 1 else 0)
    arr, keep = stv.marshal(circ.gates)
    opts = stv.options(kmax=args.kmax, tile_bits=args.tile_bits, low_bits=args.low_bits, budget=args.budget,
                       flags=args.flags, profile=True)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def one_step():
        st.set_basis(0)
        st.apply_marshalled(arr, len(circ.gates), opts)

    # a cold plan (SV_OPT_NO_PLAN_CACHE) for the record; the timed steps repeat the same
    # circuit from |0..0>, so they reuse the cached plan and its resident device blob
    st.set_basis(0)
    st.apply_marshalled(arr, len(circ.gates), stv.options(kmax=args.kmax, tile_bits=args.tile_bits,
                                                          low_bits=args.low_bits, budget=args.budget,
                                                          flags=args.flags | stv.OPT_NO_PLAN_CACHE))
    plan_cold_ms = st.stats()["plan_ms"]
    for _ in range(max(3, args.warmup)):
        one_step()
    barrier()
    tile_ms = 0.0
    flops_total = 0.0
    tile_launches = 0
    tc_flops_total = 0.0
    remap_ms = 0.0
    remap_bytes = 0.0
    launches = 0
    plan_ms = []
    kinds = {}
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            one_step()
            s = st.stats()
            tile_ms += s["pass_ms"]["tile_low"] + s["pass_ms"]["tile_high"]
            tile_launches += s["n_pass"]["tile_low"] + s["n_pass"]["tile_high"]
            launches += s["n_kernels"] + 1           # + the init kernel of set_basis
            flops_total += s["alg_flops"]
            tc_flops_total += s["tc_flops"]
            remap_ms += s["pass_ms"]["remap"]
            remap_bytes += s["remap_bytes"]
            plan_ms.append(s["plan_ms"])
            kinds = s
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    sec = ms / 1e3
    G = len(circ.gates)
    esz = 8 if args.dtype == "c64" else 16
    n_local = n - (world.bit_length() - 1)
    hbm, peak_kind = peaks()
    alg_bytes = kinds["alg_bytes"]               # per rank and circuit: 2 x esz x 2^n_local per pass
    value = alg_bytes * world / sec / 1e9        # fused-gate state-update GB/s, whole job
    gate_equiv = G * 16 * (1 << n) / sec / 1e9
    tile_bytes = 2 * esz * (1 << n_local)        # algorithmic R+W bytes per tile-pass launch
    achieved = tile_bytes / (tile_ms / max(1, tile_launches) / 1e3) / 1e9 if tile_launches else None
    # FP32 CUDA-core peak: 148 SMs x 128 FMA lanes x 2 flop x max SM clock (B200_PROFILING.md
    # unit counts; MEASURED_PEAKS.json sm_max_mhz), the ceiling of an FMA-bound tile pass
    try:
        smhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
    except Exception:
        smhz = 1965.0
    fp32_peak = 148 * 128 * 2 * smhz * 1e6 / 1e12 if args.dtype == "c64" else 148 * 64 * 2 * smhz * 1e6 / 1e12
    flops_ach = (flops_total / (tile_ms / 1e3) / 1e12) if tile_ms > 0 else None
    tc_ach = (tc_flops_total / (tile_ms / 1e3) / 1e12) if tile_ms > 0 and tc_flops_total else None
    used_tc = kinds.get("n_tc_pass", 0) > 0

    # e2e: host gate list in, full state vector out (pinned host memory)
    e2e = None
    try:   # the full-state read-back needs a pinned host copy of the state: skip it when it cannot fit
        import psutil
        host_ok = (esz << n_local) * 1.5 < psutil.virtual_memory().available
    except Exception:
        host_ok = True
    if args.e2e_steps > 0 and not host_ok:
        e2e = {"value": None, "unit": UNIT, "skipped": "pinned host copy of the %d-GiB state does not fit host RAM"
               % ((esz << n_local) >> 30)}
    if args.e2e_steps > 0 and host_ok:
        host = torch.empty((1 << n_local) * esz, dtype=torch.uint8, pin_memory=True)
        hv = host.numpy()
        ee0 = torch.cuda.Event(enable_timing=True)
        ee1 = torch.cuda.Event(enable_timing=True)
        barrier()
        ee0.record(stream)
        for _ in range(args.e2e_steps):
            st.set_basis(0)
            # no plan cache here: every e2e step plans its host gate list and copies the encoded
            # plan to the device, as a first call on a new circuit does
            st.apply(circ.gates, kmax=args.kmax, tile_bits=args.tile_bits, low_bits=args.low_bits,
                     budget=args.budget, flags=args.flags | stv.OPT_NO_PLAN_CACHE)
            if world == 1:
                st.read_state(0, 1 << n, out=hv.ctypes.data)
        ee1.record(stream)
        barrier()
        ems = ee0.elapsed_time(ee1) / args.e2e_steps
        h2d = int(st.stats().get("h2d_bytes", 0)) or None
        e2e = {"value": alg_bytes * world / (ems / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": h2d if h2d is not None else 0,
               "d2h_bytes_per_step": (esz << n) if world == 1 else 0,
               "ms_per_step": ems,
               "what": "host gate list -> sv_apply_circuit (planned from scratch, encoded plan copied H2D every step) "
                       "-> sv_read_state of all 2^n amplitudes into pinned host memory"}
        del host

    if rank != 0:
        st.close()
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        t, on, ng, note = oracle_sample(circ, args.oracle_gates, cpu_cores())
        cpu = {"value": ng * 2 * 16 * (1 << on) / t / 1e9, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
               "sample": f"first {ng} of {G} gates of {circ.name} (n={n}), complex128 gate-by-gate, "
                         f"{cpu_cores()} OpenMP threads, {t:.2f} s{note}; value = its state-update GB/s "
                         f"(each gate reads + writes the 16-B complex128 state)",
               "sec_per_circuit_extrapolated": t / ng * G * 2.0 ** (n - on)}
        # the whole c1 circuit (n=16, 380 gates) on ONE host core, for scale
        import oracle
        from inputs import circuits as Cc
        c1 = Cc.config(1)
        t1 = time.perf_counter()
        oracle.run(c1, nthreads=1)
        cpu["c1_single_core_s"] = time.perf_counter() - t1
    remap = None
    if world > 1 or remap_bytes > 0:
        remap = {"bytes_per_rank_per_step": remap_bytes / max(1, args.steps), "ms_per_step": remap_ms / max(1, args.steps),
                 "nvlink_gbs": (remap_bytes / (remap_ms / 1e3) / 1e9) if remap_ms > 0 else None}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if (world == 1 or (args.config or "ladder") == "ladder") else "strong",
        "vs_baseline": None, "dtype": "f32" if args.dtype == "c64" else "f64",
        "data": "synthetic (seeded BASELINE.json circuit; no dataset)",
        "config": {"workload": circ.name, "n": n, "gates": G, "state": args.dtype,
                   "state_bytes_per_gpu": esz << n_local, "l2": "state >> 126 MB L2 (no flush needed)",
                   "kmax": args.kmax or 4, "budget": args.budget or 1000, "tile_bits": args.tile_bits or None,
                   "flags": args.flags, "gate_kernel": "tcgen05 tensor-core" if used_tc else "CUDA-core FMA",
                   "virtual_shards": (1 << args.virtual_g) if args.virtual_g else None},
        "sec_per_circuit": sec,
        "pct_of_hbm_peak": 100.0 * value / world / hbm,
        "gate_equiv_gbs": gate_equiv,
        "passes": {k: v for k, v in kinds["n_pass"].items() if v},
        "tc_passes": kinds.get("n_tc_pass", 0), "tc_steps": kinds.get("n_tc_steps", 0),
        "ops": kinds["n_ops"],
        "plan_ms": statistics.median(plan_ms),
        "plan_cold_ms": plan_cold_ms,
        "plan_cache": "hit" if statistics.median(plan_ms) < 0.5 * plan_cold_ms else "miss",
        "gpu_launches": launches,
        "roofline": roof(used_tc, achieved, hbm, peak_kind, flops_ach, fp32_peak, tile_bytes, tile_launches, tile_ms,
                         flops_total / max(1, args.steps), tc_ach, tc_flops_total / max(1, args.steps)),
        "remap": remap,
        "clocks": clk.summary(),
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    # a plan may mix the two group-pass kernels (c3: one of its 7 passes has no operator step)
    tile_per_circuit = sum(v for k, v in kinds["n_pass"].items() if k.startswith("tile"))
    n_fma = tile_per_circuit - kinds.get("n_tc_pass", 0)   # both are counted once per pass, not per shard
    if line["roofline"] and used_tc and n_fma > 0:
        line["roofline"]["kernel"] += " + %d of %d passes per circuit on k_group_pass (CUDA-core FMA)" % (
            n_fma, tile_per_circuit)
    print(json.dumps(line), flush=True)
    st.close()


if __name__ == "__main__":
    main()
