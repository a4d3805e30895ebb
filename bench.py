"""bench.py — throughput of the QoQ W4A8 hot path on B200 (BASELINE.json metric:
"W4A8 GEMM TOPS (frac of INT8 tensor peak) and HBM GB/s at decode M, 1-8 B200").

One STEP = one decode pass of the whole hot path over all linear layers of a Llama-3-8B-shaped
model (32 layers x {qkv, o, gate, up, down}, plus a8 when N > 1), in the
paper's precision mapping (Fig. 7): per layer 4 per-token activation quantizations
(before qkv, o, gate/up, down) and 5 W4A8 GEMMs. Weights are packed offline (row a1) before timing.
The 32-layer packed weight stack (3.6 GB) is far larger than the 126 MB L2, so every step streams
weights from HBM (no flush needed).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--M 64] [--impl ours|reference]

N > 1 (torchrun): Megatron tensor parallelism — qkv/gate/up column-sharded over N (no
collective), o/down row-sharded over K at group boundaries with an NCCL all-reduce of the fp16
partials; total work is fixed ("strong" scaling).
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "W4A8 GEMM HBM GB/s at decode M (Llama-3-8B linear layers, quantizer + GEMM per step)"
UNIT = "GB/s"
FALLBACK_HBM_GBS = 6650.0          # B200_PROFILING.md fallback (used only if MEASURED_PEAKS.json is absent)
INT8_DATASHEET_TOPS = 4500.0       # dense INT8 tensor peak, datasheet


# ------------------------------------------------------------------ algorithmic work

def gemm_bytes(M, N, K):
    """What the method must move: u4 codes + s_u8/zs + s0 + q_x + s_x + t_x + Y."""
    return N * K // 2 + 2 * N * (K // 128) + 2 * N + M * K + 2 * M + 4 * M + 2 * M * N


def pc_gemm_bytes(M, N, K):
    """Per-channel W4A8 (NEXT-1): u4 codes + s_w + z_w + q_x + s_x + t_x + Y (no level-2 bytes)."""
    return N * K // 2 + 2 * N + N + M * K + 2 * M + 4 * M + 2 * M * N


def quant_bytes(M, K):
    """Per-token quantizer: read X fp16, write q_x, s_x, t_x."""
    return 2 * M * K + M * K + 2 * M + 4 * M


def rmsnorm_quant_bytes(M, K):
    """RMSNorm + per-token quantizer fused (NEXT-2): read X fp16 and gamma, write q_x, s_x, t_x."""
    return 2 * M * K + 2 * K + M * K + 2 * M + 4 * M


def silu_quant_bytes(M, I):
    """SiLU(gate)·up + per-token quantizer fused (NEXT-2): read gate and up fp16, write q_x, s_x, t_x."""
    return 4 * M * I + M * I + 2 * M + 4 * M


def gemm_ops(M, N, K):
    return 2 * M * N * K


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def load_traffic(config_key):
    """dram bytes per GEMM launch from a committed `ncu --set full` capture, if present."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(config_key)
    except Exception:
        return None


# ------------------------------------------------------------------ model layout and TP sharding

def model_shapes(model, fused=True):
    shapes, _ = synth.MODELS[model]
    return synth.fuse_gate_up(shapes) if fused else shapes


def layer_shapes(model, M, world, rank, fused=True):
    """Per-rank GEMM list of one layer: [(name, N_r, K_r, kind, quant_group)] (parallel.rank_layer_plan:
    column-parallel layers split N, a fused gate_up shard holds the rank's gate rows and up rows,
    row-parallel layers split K, both at 128 boundaries)."""
    from paper_2405_04532_b200 import parallel
    return [(name, Nr, Kr, kind, qg) for name, Nr, Kr, N, K, kind, qg in
            parallel.rank_layer_plan(model_shapes(model, fused), world)]


def step_work(model, M, layers, world, fused=True):
    """Whole-job algorithmic bytes / ops of one step (all ranks together)."""
    b = ops = 0
    for name, N, K, kind in model_shapes(model, fused):
        b += gemm_bytes(M, N, K) * layers
        ops += gemm_ops(M, N, K) * layers
    shapes = {n: (N, K) for n, N, K, _ in synth.MODELS[model][0]}
    for src in ("qkv", "o", "gate", "down"):
        b += quant_bytes(M, shapes[src][1]) * layers
    return b, ops


# ------------------------------------------------------------------ clocks during the timed region

class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index):
        self.samples = []
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _reasons(self):
        try:
            return self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            return self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append((self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM), self._reasons()))
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        mhz = [s for s, _ in self.samples]
        bits = 0
        for _, r in self.samples:
            bits |= r
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": self.max_mhz,
                "reasons": [n for b, n in self.REASONS.items() if bits & b], "samples": len(mhz)}


# ------------------------------------------------------------------ reference arm / cpu baseline (the oracle)

def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def oracle_sample(seconds_min=10.0, reps_max=200, M=64, threads=0):
    """The CPU oracle, as it stands, on a bounded sample of the workload: layer 0's o_proj
    (4096x4096, g=128) at decode M, full work (O4 quantize -> O3^-1 unpack -> level-2 dequant ->
    O5 INT32 GEMM -> O6 fp64 epilogue), repeated until >= seconds_min. threads: OpenMP threads of the
    GEMM loops (0 = all host cores). Returns (GB/s, detail)."""
    import oracle
    N, K = 4096, 4096
    W = synth.weights_fp16(N, K, seed=0)
    X = synth.activations_fp16(M, K, seed=0)
    packed, s0 = oracle.quantize_weights(W)
    all_threads = os.cpu_count() or 1
    oracle.set_num_threads(threads if threads > 0 else all_threads)
    t0 = time.perf_counter()
    reps = 0
    while reps < reps_max:
        oracle.linear_rows(X, packed, s0, N)
        reps += 1
        if time.perf_counter() - t0 >= seconds_min:
            break
    dt = time.perf_counter() - t0
    used = oracle.num_threads()
    oracle.set_num_threads(all_threads)
    b = (gemm_bytes(M, N, K) + quant_bytes(M, K)) * reps
    return b / dt / 1e9, {"reps": reps, "seconds": dt, "threads": used,
                           "sample": f"layer-0 o_proj {N}x{K} g128 at M={M}, quantize+GEMM+epilogue, x{reps}"}


def cpu_baseline_line():
    """The oracle timed on all host cores and on one core (SURVEY §8(d) "Oracle timing"), with the CPU model."""
    v, d = oracle_sample()
    v1, d1 = oracle_sample(seconds_min=4.0, threads=1)
    return {"value": v, "unit": UNIT, "cores": d["threads"], "kind": "oracle", "sample": d["sample"],
            "single_thread": {"value": v1, "unit": UNIT, "cores": 1, "sample": d1["sample"]},
            "cpu_model": cpu_model(), "host_cpus": os.cpu_count()}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    M = args.M
    N, K = 4096, 4096
    W = synth.weights_fp16(N, K, seed=0)
    X = synth.activations_fp16(M, K, seed=0)
    packed, s0 = oracle.quantize_weights(W)
    for _ in range(args.warmup):
        oracle.linear_rows(X, packed, s0, N)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.linear_rows(X, packed, s0, N)
    dt = time.perf_counter() - t0
    b = (gemm_bytes(M, N, K) + quant_bytes(M, K)) * args.steps
    v = b / dt / 1e9
    sample = f"each step: layer-0 o_proj {N}x{K} g128 at M={M} (quantize + W4A8 GEMM + epilogue) on the CPU oracle"
    cfg = config_dict(args, 1)
    cfg["workload"] = (f"{args.model} decode linear stack (reference arm: each step is a bounded sample of it, "
                       f"layer 0's o_proj {N}x{K} at M={M} with its quantizer, on the CPU oracle; GB/s of that "
                       f"sample's algorithmic bytes)")
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def config_dict(args, world):
    layers = args.layers or synth.MODELS[args.model][1]
    proj = "qkv, o, gate, up, down" if getattr(args, "unfused_gate_up", False) else "qkv, o, gate_up (fused), down"
    return {"workload": f"{args.model} decode linear stack: {layers} layers x ({proj}), "
                        f"M={args.M} tokens, W4A8 g128, per-token INT8 activations",
            "model_shapes": args.model, "M": args.M, "layers": layers, "group": 128,
            "parallelism": f"tp{world}" if world > 1 else "single",
            "activation_quant": ("fused into the GEMM prologue (qoq_w4a8_linear)"
                                 if getattr(args, "fused_quant", False) and args.M <= 64
                                 else "separate kernel (quantizer + GEMM, PDL-chained)"),
            "l2": "weights stream from HBM: packed stack >> 126 MB L2 (no flush needed)"}


# ------------------------------------------------------------------ our arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--M", type=int, default=64)
    ap.add_argument("--model", default="llama3-8b", choices=list(synth.MODELS))
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--prefill-M", type=int, default=4096)
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--no-fused-block", action="store_true")
    ap.add_argument("--no-kv4", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-streams", type=int, default=6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--detail", action="store_true", help="per-projection GEMM breakdown and M sweep")
    ap.add_argument("--no-per-channel", action="store_true",
                    help="skip the per-channel W4A8 (NEXT-1) decode step measurement")
    ap.add_argument("--unfused-gate-up", action="store_true", help="run gate and up as two GEMMs")
    ap.add_argument("--no-chain", action="store_true", help="skip the persistent decode chain measurement")
    ap.add_argument("--no-tp-fused", action="store_true",
                    help="skip the fused TP reduction leg (NEXT-3, qoq_w4a8_gemm_allreduce)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the decode M sweep (C2: M = 1 .. 256)")
    ap.add_argument("--fused-quant", action="store_true",
                    help="qoq_w4a8_linear per linear: per-token quantization fused into the GEMM prologue "
                         "(M <= 64); default: quantizer kernel + GEMM, chained with PDL (faster today)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2405_04532_b200 as qoq

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")           # communicator init (transport, NVLS) on stderr
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
    qoq.load()
    from paper_2405_04532_b200 import parallel
    M = args.M
    layers = args.layers or synth.MODELS[args.model][1]
    fused = not args.unfused_gate_up
    plan = parallel.rank_layer_plan(model_shapes(args.model, fused), world)
    shapes = [(name, Nr, Kr, kind, qg) for name, Nr, Kr, N, K, kind, qg in plan]
    stream = torch.cuda.Stream(dev)

    # ---- offline: pack every layer's FULL weights on device (row a1; the same seeded weights on every
    # rank, distinct per layer), then keep this rank's shards (parallel.shard_layer): the TP ranks hold
    # exactly the 1-GPU quantized weights
    packed = []   # [layer][i] -> (packed_r, s0_r)
    gen = torch.Generator(device=dev)
    with torch.cuda.stream(stream):
        for l in range(layers):
            full = []
            for i, (name, Nr, Kr, N, K, kind, qg) in enumerate(plan):
                gen.manual_seed(1000 * l + 17 * i)
                W = synth.device_weights_fp16(N, K, gen, dev)
                full.append(qoq.quantize_weights(W, stream=stream))
                del W
            packed.append([(p.contiguous(), s0.contiguous()) for p, s0 in parallel.shard_layer(full, plan, rank, world)])
            del full
    stream.synchronize()

    # ---- activations (L2-resident, as when produced by the preceding kernel in a real decode): one full
    # [M][K] input per quantization group, replicated on every rank; a row-parallel rank quantizes its
    # K-shard view (row stride K)
    gen.manual_seed(7)
    Kin = {}
    for name, Nr, Kr, N, K, kind, qg in plan:
        Kin[qg] = K
    X = {qg: synth.device_activations_fp16(M, K, gen, dev) for qg, K in Kin.items()}
    Kq = {qg: (Kr if kind == "row" else K) for name, Nr, Kr, N, K, kind, qg in plan}
    quant_out = {qg: (torch.empty(M, K, dtype=torch.int8, device=dev), torch.empty(M, dtype=torch.float16, device=dev),
                      torch.empty(M, dtype=torch.int32, device=dev)) for qg, K in Kq.items()}
    Ybuf = {name: torch.empty(M, N, dtype=torch.float16, device=dev) for name, N, K, kind, qg in shapes}
    ws = qoq.Workspace(dev)      # GEMM workspace (kept all-zero by the library)
    ws.get(max(qoq.gemm_workspace_bytes(M, N, K) for _, N, K, _, _ in shapes))
    lws = qoq.Workspace(dev)     # linear workspace (also holds the call's q_x / s_x / t_x)
    lws.get(max(qoq.linear_workspace_bytes(M, N, K) for _, N, K, _, _ in shapes))
    fused_quant = args.fused_quant
    if fused_quant:
        os.environ["QOQ_LINEAR_FUSED"] = "1"   # w4a8_linear's opt-in one-kernel path (read per call)

    # NEXT-3: the fused TP reduction of the row-parallel layers (qoq_w4a8_gemm_allreduce). Its buffers are
    # symmetric memory over the TP group (N > 1) or local (N = 1: the protocol's own cost, one partial)
    tp_comm, tp_comm_err = None, None
    if not args.no_tp_fused:
        n_cap = max(Nr for _, Nr, _, kind, _ in shapes if kind == "row")
        try:
            tp_comm = (parallel.fused_tp_comm(qoq, dist.group.WORLD, M, n_cap, dev) if world > 1
                       else qoq.TpComm.local(M, n_cap, dev))
        except Exception as e:   # reported in the line; the NCCL step is the measured default
            tp_comm_err = f"{type(e).__name__}: {e}"
        if world > 1:   # all ranks keep the leg, or none does
            okt = torch.tensor([0 if tp_comm is None else 1], device=dev)
            dist.all_reduce(okt, op=dist.ReduceOp.MIN)
            if not okt.item() and tp_comm is not None:
                tp_comm, tp_comm_err = None, "the fused-reduction setup failed on another rank"

    def make_linear(gemm_only, counter, fused_rows=False):
        def linear(X_r, shard, entry):
            name, Nr, Kr, N, K, kind, qg = entry
            p, s0 = shard
            if fused_rows and kind == "row":
                if not gemm_only and qg not in counter[1]:
                    qoq.quantize_activations_per_token(X_r, out=quant_out[qg], stream=stream)
                    counter[1].add(qg)
                    counter[0] += 1
                qx, sx, tx = quant_out[qg]
                qoq.w4a8_gemm_allreduce(qx, sx, tx, p, s0, Nr, tp_comm, out=Ybuf[name], stream=stream)
                counter[0] += 1
                return Ybuf[name]
            if fused_quant and not gemm_only:
                # the public linear call: per-token quantization fused into the GEMM (M <= 64)
                Xc = X_r if X_r.is_contiguous() else X_r.contiguous()
                qoq.w4a8_linear(Xc, p, s0, Nr, out=Ybuf[name], workspace=lws, stream=stream)
                counter[0] += qoq.linear_launches(M)
                return Ybuf[name]
            if not gemm_only and qg not in counter[1]:
                qoq.quantize_activations_per_token(X_r, out=quant_out[qg], stream=stream)
                counter[1].add(qg)
                counter[0] += 1
            qx, sx, tx = quant_out[qg]
            qoq.w4a8_gemm(qx, sx, tx, p, s0, Nr, out=Ybuf[name], workspace=ws, stream=stream)
            counter[0] += 1
            return Ybuf[name]
        return linear

    def run_step(gemm_only=False, collective=True, fused_rows=False):
        """One decode step: every layer through parallel.tp_decode_layer (the code path the gloo tests
        drive), the all-reduces of the row-parallel partials on `stream` — or, fused_rows, reduced inside the
        row-parallel GEMMs (NEXT-3)."""
        n_launch = 0
        for l in range(layers):
            counter = [0, set()]
            ar = (lambda Y: dist.all_reduce(Y)) if (world > 1 and collective and not gemm_only) else (lambda Y: None)
            parallel.tp_decode_layer(X, packed[l], plan, make_linear(gemm_only, counter, fused_rows), ar, rank, world,
                                     fused_rows=fused_rows)
            n_launch += counter[0]
        return n_launch

    # ---- capture one step as a CUDA graph (launch gaps removed; PDL edges kept)
    with torch.cuda.stream(stream):
        run_step()
        run_step(gemm_only=True)
    stream.synchronize()
    g_step = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_step, stream=stream):
        launches_per_step = run_step()
    g_gemm = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_gemm, stream=stream):
        gemm_launches = run_step(gemm_only=True)
    g_nocoll = None
    if world > 1:
        g_nocoll = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_nocoll, stream=stream):
            run_step(collective=False)

    def timed(graph, steps, warmup):
        for _ in range(warmup):
            graph.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            graph.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    with torch.cuda.stream(stream):
        sampler = ClockSampler(local)
        for _ in range(args.warmup):
            g_step.replay()
        with sampler:
            ms_total = timed(g_step, args.steps, 0)
        ms_gemm = timed(g_gemm, max(10, args.steps // 2), 2)
        ms_nocoll = timed(g_nocoll, max(10, args.steps // 2), 2) / max(10, args.steps // 2) if g_nocoll else None

    # ---- NEXT-3: the same step with the row-parallel reductions fused into the GEMM epilogues. One eager step
    # first: a peer wait that timed out (status) or outputs outside the propagated tolerance of the NCCL step
    # disable the timed leg instead of timing a broken protocol. N = 1: the protocol's own cost per launch on
    # the TP = 8 row-parallel shard shapes (the one-partial reduction against the plain GEMM)
    tp_fused = None
    if tp_comm is not None and world == 1:
        try:
            tp_fused = tp_fused_overhead(qoq, torch, args, dev, stream, timed)
        except Exception as e:
            tp_fused = {"unavailable": f"{type(e).__name__}: {e}"}
    elif tp_comm is not None:
        try:
            with torch.cuda.stream(stream):
                run_step()
                ref_rows = {n: Ybuf[n].clone() for n, _, _, kind, _ in shapes if kind == "row"}
                run_step(fused_rows=True)
            stream.synchronize()
            if world > 1:
                dist.barrier()
            st = tp_comm.status()
            diff = max(float((Ybuf[n].float() - ref_rows[n].float()).abs().max()) for n in ref_rows)
            scale = max(float(ref_rows[n].float().abs().max()) for n in ref_rows)
            ok = st == 0 and diff <= 4e-3 * scale + 2e-3 * world
            # every rank takes the same branch (the timed leg has barriers / all-reduces): ok on ALL ranks
            okt = torch.tensor([1 if ok else 0], device=dev)
            dist.all_reduce(okt, op=dist.ReduceOp.MIN)
            ok = bool(okt.item())
            tp_fused = {"status": st, "max_abs_diff_vs_nccl_step": diff, "ok": ok}
            if ok:
                g_fused = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g_fused, stream=stream):
                    run_step(fused_rows=True)
                with torch.cuda.stream(stream):
                    nst = max(10, args.steps // 2)
                    ms_f = timed(g_fused, nst, 2) / nst
                tp_fused.update({"ms_per_step": ms_f, "GBps": step_work(args.model, M, layers, world, fused)[0]
                                 / (ms_f * 1e-3) / 1e9, "status_after": tp_comm.status()})
        except Exception as e:
            tp_fused = {"unavailable": f"{type(e).__name__}: {e}"}
        tp_fused["what"] = ("decode step with the row-parallel all-reduces fused into the o / down GEMM epilogues "
                            "(qoq_w4a8_gemm_allreduce: fp16 partial tiles pushed to every rank's symmetric buffer, "
                            "reduced in rank order, NEXT-3)")
    elif tp_comm_err:
        tp_fused = {"unavailable": tp_comm_err}

    ms_step = ms_total / args.steps
    step_bytes, step_ops = step_work(args.model, M, layers, world, fused)
    value = step_bytes / (ms_step * 1e-3) / 1e9

    # dominant kernel: the W4A8 GEMM. Fused (M <= 64): every launch of the step is the GEMM kernel with
    # the quantization in its prologue, so its per-launch figures come from the step; two-kernel: the
    # GEMM-only graph.
    if fused_quant and qoq.linear_launches(M) == 1:
        rank_gemm_bytes = sum(gemm_bytes(M, N, K) + quant_bytes(M, K) for _, N, K, _, _ in shapes) * layers
        per_launch_ms = ms_step / launches_per_step
        per_launch_bytes = rank_gemm_bytes / launches_per_step
        kernel_name = "w4a8_gemm_kernel (per-token quantization fused)"
    else:
        rank_gemm_bytes = sum(gemm_bytes(M, N, K) for _, N, K, _, _ in shapes) * layers
        per_launch_ms = ms_gemm / max(10, args.steps // 2) / gemm_launches
        per_launch_bytes = rank_gemm_bytes / gemm_launches
        kernel_name = "w4a8_gemm_kernel"
    achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
    peak, peak_src = load_peaks()
    traffic = load_traffic(f"{args.model}-M{M}" + ("-fused" if kernel_name != "w4a8_gemm_kernel" else ""))
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": kernel_name,
                "algorithmic_bytes_per_launch": per_launch_bytes, "avg_launch_us": per_launch_ms * 1e3,
                "peak_source": peak_src}
    tops = step_ops / (ms_step * 1e-3) / 1e12

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "int8",
            "data": "synthetic (seeded N(0,1/K) fp16 weights packed on device; N(0,1) fp16 activations "
                    "with 0.1% x20 outlier channels)",
            "config": config_dict(args, world), "gpu_launches": launches_per_step * args.steps,
            "clocks": sampler.summary(), "roofline": roofline,
            "decode_tops": tops, "decode_frac_int8_datasheet": tops / INT8_DATASHEET_TOPS}
    if world > 1:
        # eta_TP = T_roofline,1GPU(full step) / (TP x T_measured,rank), with and without the
        # all-reduces of the row-parallel partials
        t_roof = step_bytes / (peak * 1e9) * 1e3
        line["tp"] = {"world": world, "ms_per_step": ms_step, "ms_per_step_no_collective": ms_nocoll,
                      "ms_gemm_only": ms_gemm / max(10, args.steps // 2),
                      "eta_with_collective": t_roof / (world * ms_step),
                      "eta_no_collective": t_roof / (world * ms_nocoll) if ms_nocoll else None,
                      "t_roofline_1gpu_ms": t_roof,
                      "collective": "torch.distributed.all_reduce (NCCL) of the fp16 row-parallel partials"}

    if tp_fused is not None:
        line["tp_fused"] = tp_fused
    if world == 1 and not args.no_chain and M <= 128:
        line["decode_chain"] = chain_measure(qoq, torch, args, plan, packed, layers, dev, stream, X, step_bytes, timed)
    if world == 1 and not args.no_sweep:
        line["decode_sweep"] = sweep_measure(qoq, torch, args, plan, packed, layers, dev, stream, timed)

    # ---- per-channel W4A8 (NEXT-1, §5.2.2): the same decode step on per-channel packed weights
    if not args.no_per_channel and world == 1:
        line["per_channel"] = per_channel_measure(qoq, torch, args, shapes, layers, dev, stream, X, quant_out,
                                                  Ybuf, ws, timed)

    # ---- the paper's block mapping (Fig. 7): quantization fused into RMSNorm / SiLU·mul (NEXT-2)
    if not args.no_fused_block and world == 1:
        line["fused_block"] = fused_block_measure(qoq, torch, args, shapes, packed, layers, dev, stream, X,
                                                  quant_out, Ybuf, ws, timed)

    # ---- KV4 decode attention (NEXT-4, §5.3): the paper's other hot kernel, Llama-3-8B heads
    if not args.no_kv4 and world == 1:
        line["kv4_attention"] = kv4_measure(qoq, torch, dev, stream, timed)

    # ---- e2e through the C ABI with host buffers (H2D + quantize + GEMM + D2H per GEMM)
    if not args.no_e2e:
        # N > 1: one stream, so every rank issues its all-reduces in one order (collectives spread over
        # several streams may interleave differently across ranks and deadlock)
        line["e2e"] = e2e_measure(qoq, torch, dist, args, shapes, packed, layers, world, dev, stream, step_bytes,
                                  nstreams=args.e2e_streams if world == 1 else 1)

    if not args.no_prefill:
        line["prefill"] = prefill_measure(qoq, torch, args, shapes, packed, layers, dev, stream)
        if world == 1:
            # the >= 1024 side of the north_star target (C3 at 4096 / 8192 plus 1024 / 2048)
            sweep = {}
            for Mp in (1024, 2048, 4096, 8192):
                r = prefill_measure(qoq, torch, args, shapes, packed, layers, dev, stream, M=Mp, with_ceiling=False)
                sweep[str(Mp)] = {k: r[k] for k in ("tops", "ms", "frac_int8_datasheet", "per_gemm_tops")}
                sweep[str(Mp)]["frac_int8_measured_ceiling"] = (r["tops"] / line["prefill"]["int8_ceiling_tops"]
                                                                 if line["prefill"]["int8_ceiling_tops"] else None)
            line["prefill"]["sweep"] = sweep

    if args.detail:
        line["detail"] = detail_measure(qoq, torch, args, shapes, packed, layers, dev, stream, X)

    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_line()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line))
    return 0


def e2e_measure(qoq, torch, dist, args, shapes, packed, layers, world, dev, stream, step_bytes, nstreams=6):
    """End to end through the C ABI (qoq_linear_host: pinned host X -> device -> w4a8_linear ->
    pinned host Y) for every GEMM of the step. Consecutive calls alternate over `nstreams` CUDA
    streams (each with its own scratch and host buffers), so one call's D2H copy overlaps the next
    call's H2D copy and kernels (PCIe is full duplex); every copy of the step stays in the timed
    region."""
    M = args.M
    gen = torch.Generator().manual_seed(3)
    streams = [stream] + [torch.cuda.Stream(dev) for _ in range(nstreams - 1)]
    Xh, Yh, scratch, red = {}, {}, {}, {}
    for j in range(nstreams):
        for name, N, K, kind, qg in shapes:
            Xh[j, name] = (torch.randn(M, K, generator=gen) * 1.0).half().pin_memory()
            Yh[j, name] = torch.empty(M, N, dtype=torch.float16).pin_memory()
            # one scratch per (stream, projection shape): the header's workspace-reuse rule
            scratch[j, name] = torch.zeros(qoq.linear_host_scratch_bytes(M, N, K), dtype=torch.uint8, device=dev)
            if kind == "row":
                red[j, name] = torch.empty(M, N, dtype=torch.float16, device=dev)
    h2d = sum(M * K * 2 for _, N, K, _, _ in shapes) * layers
    d2h = sum(M * N * 2 for _, N, K, _, _ in shapes) * layers

    def one_step():
        c = 0
        for l in range(layers):
            for i, (name, N, K, kind, qg) in enumerate(shapes):
                j = c % nstreams
                c += 1
                st = streams[j]
                p, s0 = packed[l][i]
                qoq.linear_host(Xh[j, name], p, s0, N, Yh[j, name], scratch[j, name], stream=st)
                if kind == "row" and world > 1:
                    with torch.cuda.stream(st):
                        red[j, name].copy_(Yh[j, name], non_blocking=True)
                        dist.all_reduce(red[j, name])
                        Yh[j, name].copy_(red[j, name], non_blocking=True)

    def forked_step():
        """one_step with the side streams forked from / joined into streams[0] (graph capture)."""
        ev0 = torch.cuda.Event()
        ev0.record(streams[0])
        for st in streams[1:]:
            st.wait_event(ev0)
        one_step()
        for st in streams[1:]:
            ev = torch.cuda.Event()
            ev.record(st)
            streams[0].wait_event(ev)

    steps = max(3, args.steps // 10)
    for _ in range(2):
        forked_step()
    torch.cuda.synchronize(dev)
    # the step's API calls (copies + kernels of all 4 x layers linear_host calls) captured once as a
    # CUDA graph and replayed: no per-call host overhead in the timed region, every copy still in it
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=streams[0]):
        forked_step()
    g.replay()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(streams[0]):
        e0.record(streams[0])
        for _ in range(steps):
            g.replay()
        e1.record(streams[0])
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": step_bytes / (ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d * world,
            "d2h_bytes_per_step": d2h * world, "ms_per_step": ms, "steps": steps, "streams": nstreams,
            "api": "qoq_linear_host (C ABI, pinned host X/Y) per GEMM, calls alternating over "
                   f"{nstreams} streams, the step captured as one CUDA graph"}


def tp_fused_overhead(qoq, torch, args, dev, stream, timed, world_tp=8, reps=16):
    """NEXT-3 at N = 1: per-launch time of qoq_w4a8_gemm_allreduce with a one-rank comm (push, flag, wait and
    rank-order reduction all local) against qoq_w4a8_gemm on the row-parallel shard shapes of TP = world_tp
    (o: K / world_tp, down: I / world_tp), graphs of `reps` distinct weights each."""
    M = args.M
    gen = torch.Generator(device=dev)
    out = {}
    for name, N, K, kind in model_shapes(args.model, True):
        if kind != "row":
            continue
        Kr = K // world_tp
        packs = []
        for i in range(reps):
            gen.manual_seed(9000 + i)
            packs.append(qoq.quantize_weights(synth.device_weights_fp16(N, Kr, gen, dev), stream=stream))
        qx, sx, tx = qoq.quantize_activations_per_token(synth.device_activations_fp16(M, Kr, gen, dev), stream=stream)
        Y = torch.empty(M, N, dtype=torch.float16, device=dev)
        comm = qoq.TpComm.local(M, N, dev)
        ws = qoq.Workspace(dev)
        ws.get(qoq.gemm_workspace_bytes(M, N, Kr))
        res = {}
        for leg in ("gemm", "fused"):
            def run():
                for p, s0 in packs:
                    if leg == "gemm":
                        qoq.w4a8_gemm(qx, sx, tx, p, s0, N, out=Y, workspace=ws, stream=stream)
                    else:
                        qoq.w4a8_gemm_allreduce(qx, sx, tx, p, s0, N, comm, out=Y, stream=stream)
            with torch.cuda.stream(stream):
                run()
            stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                run()
            with torch.cuda.stream(stream):
                res[leg + "_us"] = timed(g, 20, 3) / 20 / reps * 1e3
        res["status"] = comm.status()
        out[f"{name}_N{N}_K{Kr}"] = res
    return {"per_launch": out, "M": M, "tp_shard_of": world_tp,
            "what": "N = 1: qoq_w4a8_gemm_allreduce with a one-rank comm (the fused reduction's own cost: local "
                    "flag-in-data push and rank-order reduce) vs qoq_w4a8_gemm, on the TP = 8 "
                    "row-parallel shard shapes; the cross-GPU leg runs under torchrun (N > 1)"}


def chain_measure(qoq, torch, args, plan, packed, layers, dev, stream, X, step_bytes, timed):
    """The same decode step through the persistent decode chain (qoq_w4a8_linear_chain): every linear of
    the stack in ONE launch per <= 128 linears, the per-token quantization inside the kernel, each linear
    waiting for the previous one's output (the sequential dependency of a real decode)."""
    M = args.M
    Y = {name: torch.empty(M, N, dtype=torch.float16, device=dev) for name, Nr, Kr, N, K, kind, qg in plan}
    lin = []
    for l in range(layers):
        for (p, s0), (name, Nr, Kr, N, K, kind, qg) in zip(packed[l], plan):
            lin.append((X[qg], p, s0, N, Y[name], K))
    chunks = [lin[i:i + 128] for i in range(0, len(lin), 128)]
    ws = qoq.Workspace(dev)

    def run():
        for c in chunks:
            qoq.w4a8_linear_chain(c, workspace=ws, stream=stream)

    with torch.cuda.stream(stream):
        run()
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            run()
        steps = max(10, args.steps // 2)
        ms = timed(g, steps, 3) / steps
    del Y
    return {"value": step_bytes / (ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms, "launches_per_step": len(chunks),
            "what": "same decode step in one persistent kernel per <= 128 linears (qoq_w4a8_linear_chain): "
                    "in-kernel per-token quantization, k-split / stream-K over all SMs, grid-wide ordering"}


def sweep_measure(qoq, torch, args, plan, packed, layers, dev, stream, timed, Ms=(1, 2, 4, 8, 16, 32, 64, 128, 256)):
    """BASELINE config C2: the decode step (quantizer + W4A8 GEMM per linear, one CUDA graph) over the
    decode token counts M = 1 .. 256, GB/s of the §8(d) algorithmic bytes and TOPS."""
    out = {}
    gen = torch.Generator(device=dev)
    for M in (Ms[0],) + tuple(Ms):          # the first configuration twice: the first pass only warms up
        gen.manual_seed(70 + M)
        Xs = {}
        for name, Nr, Kr, N, K, kind, qg in plan:
            Xs[qg] = synth.device_activations_fp16(M, K, gen, dev)
        qo = {qg: (torch.empty(M, x.shape[1], dtype=torch.int8, device=dev), torch.empty(M, dtype=torch.float16, device=dev),
                   torch.empty(M, dtype=torch.int32, device=dev)) for qg, x in Xs.items()}
        Ys = {name: torch.empty(M, Nr, dtype=torch.float16, device=dev) for name, Nr, Kr, N, K, kind, qg in plan}
        wsm = qoq.Workspace(dev)
        wsm.get(max(qoq.gemm_workspace_bytes(M, Nr, Kr) for name, Nr, Kr, N, K, kind, qg in plan))

        def run():
            for l in range(layers):
                done = set()
                for (p, s0), (name, Nr, Kr, N, K, kind, qg) in zip(packed[l], plan):
                    if qg not in done:
                        qoq.quantize_activations_per_token(Xs[qg], out=qo[qg], stream=stream)
                        done.add(qg)
                    qx, sx, tx = qo[qg]
                    qoq.w4a8_gemm(qx, sx, tx, p, s0, Nr, out=Ys[name], workspace=wsm, stream=stream)

        with torch.cuda.stream(stream):
            run()
            stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                run()
            steps = 10
            ms = timed(g, steps, 3) / steps
        nb, ops = step_work(args.model, M, layers, 1, not args.unfused_gate_up)
        out[str(M)] = {"ms_per_step": ms, "GBps": nb / (ms * 1e-3) / 1e9, "TOPS": ops / (ms * 1e-3) / 1e12}
        del g, Xs, qo, Ys
    return out


def per_channel_measure(qoq, torch, args, shapes, layers, dev, stream, X, quant_out, Ybuf, ws, timed):
    """The decode step with per-channel W4A8 weights (quantizer + qoq_pc_w4a8_gemm per projection),
    captured as one CUDA graph like the main step; GB/s over the per-channel algorithmic bytes."""
    M = args.M
    gen = torch.Generator(device=dev)
    pcs = []
    with torch.cuda.stream(stream):
        for l in range(layers):
            row = []
            for i, (name, N, K, kind, qg) in enumerate(shapes):
                gen.manual_seed(1000 * l + 17 * i)
                W = synth.device_weights_fp16(N, K, gen, dev)
                row.append(qoq.pc_quantize_weights(W, stream=stream))
                del W
            pcs.append(row)
    stream.synchronize()

    def run():
        for l in range(layers):
            done = set()
            for i, (name, N, K, kind, qg) in enumerate(shapes):
                if qg not in done:
                    qoq.quantize_activations_per_token(X[qg], out=quant_out[qg], stream=stream)
                    done.add(qg)
                qx, sx, tx = quant_out[qg]
                p, s_w, z_w = pcs[l][i]
                qoq.pc_w4a8_gemm(qx, sx, tx, p, s_w, z_w, N, out=Ybuf[name], workspace=ws, stream=stream)

    with torch.cuda.stream(stream):
        run()
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            run()
        steps = max(10, args.steps // 2)
        ms = timed(g, steps, 3) / steps
    b = 0
    for name, N, K, kind, qg in shapes:
        b += pc_gemm_bytes(M, N, K) * layers
    shp = {n: (N, K) for n, N, K, _ in synth.MODELS[args.model][0]}
    for src in ("qkv", "o", "gate", "down"):
        b += quant_bytes(M, shp[src][1]) * layers
    del pcs
    return {"value": b / (ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms, "steps": steps,
            "what": "same decode step, per-channel W4A8 weights (qoq_pc_w4a8_gemm, NEXT-1)"}


def fused_block_measure(qoq, torch, args, shapes, packed, layers, dev, stream, X, quant_out, Ybuf, ws, timed):
    """The decode step with the activation quantization of Fig. 7: RMSNorm+quantize before qkv
    and gate_up, the separate quantizer before o, SiLU·mul+quantize (on the gate_up GEMM's own output)
    before down — one CUDA graph; plus each fused quantizer timed alone at decode M and prefill M
    (inputs rotated over > L2 bytes) against the HBM peak."""
    M = args.M
    gen = torch.Generator(device=dev)
    gen.manual_seed(23)
    Kh = {qg: K for _, N, K, _, qg in shapes}
    I = Kh["mlp_act"]
    gam = [(1.0 + 0.1 * torch.randn(2, Kh["attn_in"], generator=gen, device=dev)).half() for _ in range(layers)]
    eps = 1e-5

    def run():
        n = 0
        for l in range(layers):
            for i, (name, N, K, kind, qg) in enumerate(shapes):
                if qg == "attn_in":
                    qoq.rmsnorm_quantize(X[qg], gam[l][0], eps, out=quant_out[qg], stream=stream)
                elif qg == "mlp_in":
                    qoq.rmsnorm_quantize(X[qg], gam[l][1], eps, out=quant_out[qg], stream=stream)
                elif qg == "mlp_act":
                    qoq.silu_mul_quantize(Ybuf["gate_up"], out=quant_out[qg], stream=stream)
                else:
                    qoq.quantize_activations_per_token(X[qg], out=quant_out[qg], stream=stream)
                qx, sx, tx = quant_out[qg]
                p, s0 = packed[l][i]
                qoq.w4a8_gemm(qx, sx, tx, p, s0, N, out=Ybuf[name], workspace=ws, stream=stream)
                n += 2
        return n

    with torch.cuda.stream(stream):
        run()
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            launches = run()
        steps = max(10, args.steps // 2)
        ms = timed(g, steps, 3) / steps
    b = sum(gemm_bytes(M, N, K) for _, N, K, _, _ in shapes) * layers
    b += (2 * rmsnorm_quant_bytes(M, Kh["attn_in"]) + quant_bytes(M, Kh["attn_out"]) + silu_quant_bytes(M, I)) * layers
    out = {"value": b / (ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms, "steps": steps,
           "launches_per_step": launches,
           "what": "decode step with Fig. 7's quantization mapping: rmsnorm_quantize -> qkv, quantize -> o, "
                   "rmsnorm_quantize -> gate_up, silu_mul_quantize(gate_up output) -> down (NEXT-2)"}
    peak, _ = load_peaks()
    kern = {}
    for Mk in (M, args.prefill_M):
        for kname, K, nbytes in (("rmsnorm_quant_kernel", Kh["attn_in"], rmsnorm_quant_bytes(Mk, Kh["attn_in"])),
                                 ("silu_mul_quant_kernel", I, silu_quant_bytes(Mk, I))):
            in_bytes = (2 if kname.startswith("rms") else 4) * Mk * K
            nbuf = max(1, min(8, -(-256 * 2 ** 20 // in_bytes)))     # rotate inputs over >= 256 MB (> L2)
            if kname.startswith("rms"):
                ins = [synth.device_activations_fp16(Mk, K, gen, dev) for _ in range(nbuf)]
            else:
                ins = [(2.0 * torch.randn(Mk, 2 * K, generator=gen, device=dev)).half() for _ in range(nbuf)]
            o = (torch.empty(Mk, K, dtype=torch.int8, device=dev), torch.empty(Mk, dtype=torch.float16, device=dev),
                 torch.empty(Mk, dtype=torch.int32, device=dev))
            reps = 4 * nbuf if Mk > M else 64

            def krun():
                for r in range(reps):
                    if kname.startswith("rms"):
                        qoq.rmsnorm_quantize(ins[r % nbuf], gam[0][0], eps, out=o, stream=stream)
                    else:
                        qoq.silu_mul_quantize(ins[r % nbuf], out=o, stream=stream)

            with torch.cuda.stream(stream):
                krun()
                stream.synchronize()
                gk = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gk, stream=stream):
                    krun()
                us = timed(gk, 5, 2) / 5 / reps * 1e3
            kern[f"{kname}_M{Mk}"] = {"K": K, "us": us, "GBps": nbytes / (us * 1e-6) / 1e9,
                                      "frac_hbm": nbytes / (us * 1e-6) / 1e9 / peak,
                                      "algorithmic_bytes": nbytes}
            del ins, o
    out["kernels"] = kern
    return out


def kv4_measure(qoq, torch, dev, stream, timed, B=64, T=1024, H=32, H_kv=8, D=128, P=64, layers=4):
    """Decode attention over a paged KV4 cache (qoq_kv4_decode_attention): B sequences x T tokens,
    Llama-3-8B heads, one call per layer over `layers` distinct caches (> L2 in total). Algorithmic bytes
    per call: the cache (K + V codes D bytes + 8 bytes of fp16 scale/zero per token and kv head), Q, O and
    the block table. The cache is filled on the device with qoq_kv4_append from seeded normals."""
    gen = torch.Generator(device=dev)
    gen.manual_seed(31)
    npg = T // P
    pb = qoq.kv4_page_bytes(H_kv, D, P)
    caches = []
    with torch.cuda.stream(stream):
        for l in range(layers):
            pages = torch.zeros(B * npg * pb, dtype=torch.uint8, device=dev)
            bt = torch.randperm(B * npg, generator=gen, device=dev).to(torch.int32).view(B, npg)
            for t in range(T):
                Kt = torch.randn(B, H_kv, D, generator=gen, device=dev).half()
                Vt = torch.randn(B, H_kv, D, generator=gen, device=dev).half()
                slots = (bt[:, t // P] * P + t % P).contiguous()
                qoq.kv4_append(Kt, Vt, slots, pages, P, stream=stream)
            caches.append((pages, bt))
        lens = torch.full((B,), T, dtype=torch.int32, device=dev)
        Q = torch.randn(B, H, D, generator=gen, device=dev).half()
        O = torch.empty_like(Q)
        stream.synchronize()

        def run():
            for pages, bt in caches:
                qoq.kv4_decode_attention(Q, pages, bt, lens, H_kv, P, out=O, stream=stream)

        run()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            run()
        reps = 10
        us = timed(g, reps, 3) / reps / layers * 1e3
    nbytes = B * T * H_kv * (D + 8) + 2 * 2 * B * H * D + 4 * B * npg + 4 * B
    peak, _ = load_peaks()
    gbps = nbytes / (us * 1e-6) / 1e9
    return {"us": us, "GBps": gbps, "frac_hbm": gbps / peak, "algorithmic_bytes": nbytes,
            "config": {"B": B, "seq_len": T, "H": H, "H_kv": H_kv, "D": D, "page_size": P, "layers_rotated": layers},
            "paper_context": "A100 QServe KV4 kernel 0.28 ms at seq 1024 (Table P:507-526; other GPU/model: context only)"}


def prefill_measure(qoq, torch, args, shapes, packed, layers, dev, stream, M=None, with_ceiling=True):
    """Tensor-bound regime (BASELINE configs[2]): GEMM-only TOPS at M = prefill_M over the first
    4 layers' weights (rotating, > L2), per projection, and the INT8 ceiling measured with cuBLASLt in
    the same run."""
    M = args.prefill_M if M is None else M
    L = min(4, layers)
    gen = torch.Generator(device=dev)
    gen.manual_seed(11)
    Ks = sorted({K for _, N, K, _, _ in shapes})
    q = {}
    for K in Ks:
        Xp = synth.device_activations_fp16(M, K, gen, dev)
        q[K] = qoq.quantize_activations_per_token(Xp, stream=stream)
    Y = {name: torch.empty(M, N, dtype=torch.float16, device=dev) for name, N, K, kind, qg in shapes}
    ws = qoq.Workspace(dev)

    def run():
        for l in range(L):
            for i, (name, N, K, kind, qg) in enumerate(shapes):
                qx, sx, tx = q[K]
                p, s0 = packed[l][i]
                qoq.w4a8_gemm(qx, sx, tx, p, s0, N, out=Y[name], workspace=ws, stream=stream)

    with torch.cuda.stream(stream):
        run()
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            run()
        for _ in range(3):
            g.replay()
        stream.synchronize()
        reps = 5
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
        stream.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ops = sum(gemm_ops(M, N, K) for _, N, K, _, _ in shapes) * L
    tops = ops / (ms * 1e-3) / 1e12
    per = {}
    with torch.cuda.stream(stream):   # each projection alone (rotating over the L layers' weights)
        for i, (name, N, K, kind, qg) in enumerate(shapes):
            qx, sx, tx = q[K]

            def one():
                for l in range(L):
                    p, s0 = packed[l][i]
                    qoq.w4a8_gemm(qx, sx, tx, p, s0, N, out=Y[name], workspace=ws, stream=stream)

            one()
            g1 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g1, stream=stream):
                one()
            g1.replay()
            stream.synchronize()
            e0.record(stream)
            for _ in range(reps):
                g1.replay()
            e1.record(stream)
            stream.synchronize()
            t1 = e0.elapsed_time(e1) / reps / L
            per[name] = gemm_ops(M, N, K) / (t1 * 1e-3) / 1e12
    ceil = int8_ceiling(torch, dev) if with_ceiling else None
    del q, Y
    return {"M": M, "layers": L, "tops": tops, "ms": ms, "per_gemm_tops": per,
            "frac_int8_datasheet": tops / INT8_DATASHEET_TOPS,
            "int8_ceiling_tops": ceil, "frac_int8_measured_ceiling": tops / ceil if ceil else None,
            "ceiling_how": "torch._int_mm (cuBLASLt IMMA) 8192^3 best of 10, same run"}


def int8_ceiling(torch, dev):
    try:
        a = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device=dev)
        b = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device=dev).t()
        torch._int_mm(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return 2 * 8192 ** 3 / (best * 1e-3) / 1e12
    except Exception:
        return None


def detail_measure(qoq, torch, args, shapes, packed, layers, dev, stream, X):
    out = {}
    M = args.M
    for i, (name, N, K, kind, qg) in enumerate(shapes):
        qx, sx, tx = qoq.quantize_activations_per_token(X[qg], stream=stream)
        Y = torch.empty(M, N, dtype=torch.float16, device=dev)
        ws = qoq.Workspace(dev)

        def run():
            for l in range(layers):
                p, s0 = packed[l][i]
                qoq.w4a8_gemm(qx, sx, tx, p, s0, N, out=Y, workspace=ws, stream=stream)

        with torch.cuda.stream(stream):
            run()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                run()
            for _ in range(3):
                g.replay()
            stream.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(10):
                g.replay()
            e1.record(stream)
            stream.synchronize()
        us = e0.elapsed_time(e1) / 10 / layers * 1e3
        out[name] = {"N": N, "K": K, "us": us, "GBps": gemm_bytes(M, N, K) / (us * 1e-6) / 1e9}
    return out


if __name__ == "__main__":
    sys.exit(main())
