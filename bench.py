#!/usr/bin/env python3
"""SBVR GEMV benchmark on B200 (BASELINE.json metric: SBVR GEMV HBM GB/s and us/GEMV vs fp16 cuBLAS).

One step = the decode hot path of one Llama-3-8B decoder layer at batch 1 (BASELINE.json configs[1]):
    4 activation conversions (sbvr_encode_vector, Eq. 12) + 7 SBVR GEMVs (sbvr_gemv, W4A8, §4.4)
    for q/k/v/o (4096x4096, 1024x4096 x2, 4096x4096), gate/up (14336x4096 x2), down (4096x14336).
Steps cycle through a ring of distinct layer weight sets (4 x 117 MB > 126 MB L2), each step is one
CUDA-graph replay; device time is measured with CUDA events, max over ranks.  At N > 1 every matrix is
row-sharded over the ranks and each GEMV is followed by an NCCL all-gather of y (total work fixed).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synthetic  # noqa: E402
from paper_2509_18172_b200 import dist as sdist  # noqa: E402

METRIC = "SBVR GEMV HBM GB/s (% of 8 TB/s) and µs/GEMV at 1/2/4/8 B200 vs fp16 cuBLAS"
K_BITS, L_BITS, G, N_RATIO = 4, 8, 128, 16
EV_EVERY = 32         # one timed step in EV_EVERY carries the CUDA-event span around its GEMV launches (roofline)
# which activation feeds which projection: q,k,v <- x_attn; o <- x_o; gate,up <- x_mlp; down <- x_down
INPUT_OF = {"q_proj": 0, "k_proj": 0, "v_proj": 0, "o_proj": 1, "gate_proj": 2, "up_proj": 2, "down_proj": 3}
INPUT_N = [4096, 4096, 4096, 14336]


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ------------------------------------------------------------------ CUDA runtime helpers (external event nodes)
class _Cudart:
    def __init__(self):
        self.lib = ctypes.CDLL("libcudart.so.12")
        self.lib.cudaEventCreateWithFlags.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_uint]
        self.lib.cudaEventRecordWithFlags.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint]
        self.lib.cudaEventSynchronize.argtypes = [ctypes.c_void_p]
        self.lib.cudaEventElapsedTime.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.c_void_p, ctypes.c_void_p]

    def event(self):
        ev = ctypes.c_void_p()
        assert self.lib.cudaEventCreateWithFlags(ctypes.byref(ev), 0) == 0
        return ev

    def record_external(self, ev, stream):
        # cudaEventRecordExternal (0x1): inside stream capture this becomes an event-record node
        assert self.lib.cudaEventRecordWithFlags(ev, ctypes.c_void_p(stream.cuda_stream), 1) == 0

    def elapsed_ms(self, a, b):
        assert self.lib.cudaEventSynchronize(b) == 0
        ms = ctypes.c_float()
        assert self.lib.cudaEventElapsedTime(ctypes.byref(ms), a, b) == 0
        return ms.value


# ------------------------------------------------------------------ clocks sampler (NVML, during the loaded region)
class ClockSampler:
    """Samples SM clock, power and clock-event (throttle) reasons through NVML every `interval_s` from a
    host thread while the GPU runs the heat-up and the timed steps (the timed region alone can be ~1 ms
    at --steps 20, shorter than nvidia-smi's sampling period; NVML is polled directly)."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, local_rank: int, interval_s: float = 0.001):
        self.rows, self.h, self.max_sm = [], None, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            ids = [v for v in vis.split(",") if v.strip()]
            idx = int(ids[local_rank]) if ids and all(v.strip().isdigit() for v in ids) else local_rank
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, args=(interval_s,), daemon=True)
            self.t.start()
        except Exception:
            self.h = None

    def _run(self, dt):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                self.rows.append((time.time(), sm, rs, pw))
            except Exception:
                pass
            time.sleep(dt)

    def stop(self):
        self._stop.set()
        if self.h is not None:
            self.t.join(timeout=2)

    def summary(self, t0: float, t1: float):
        rows = [r for r in self.rows if t0 <= r[0] <= t1 + 0.002]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_sm, "reasons": [], "samples": 0}
        reasons = sorted({n for _, _, rs, _ in rows for bit, n in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(r[1] for r in rows), "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": len(rows), "sm_mhz_min": min(r[1] for r in rows), "power_w_max": max(r[3] for r in rows),
                "window": "NVML, 1 ms period, over the clock heat-up and the timed steps"}


# ------------------------------------------------------------------ workload
def layer_shapes():
    """The 7 projections of one Llama-3-8B decoder layer (name, M, N)."""
    return list(synthetic.LLAMA3_8B_LAYER)


# As deployed (vLLM QKVParallelLinear / MergedColumnParallelLinear): projections that read the same
# input are one matrix with their rows stacked.  (name, M, N, input index, member projections)
FUSED = [("qkv_proj", 6144, 4096, 0, ("q_proj", "k_proj", "v_proj")), ("o_proj", 4096, 4096, 1, ("o_proj",)),
         ("gate_up_proj", 28672, 4096, 2, ("gate_proj", "up_proj")), ("down_proj", 4096, 14336, 3, ("down_proj",))]


def build_ring(sb, ring, world, rank, device):
    """Ring of `ring` distinct layers of fused matrices; each matrix row-sharded to this rank."""
    layers = []
    for r in range(ring):
        mats = []
        for idx, (name, M, N, xin, _) in enumerate(FUSED):
            r0, r1 = sdist.shard_range(M, world, rank)
            pc, s16, b16, ri = synthetic.random_encoded(r1 - r0, N, K_BITS, N_RATIO, seed=400 + 7 * r + idx + 1000 * rank)
            w = sb.pack_canonical(pc, s16, b16, ri, N_RATIO, device=device)
            mats.append((name, M, N, r0, r1, w, sb.Workspace.for_weights(w, 1), xin))
        layers.append(mats)
    return layers


def gemv_bytes(sb, M, N):
    return sb.algorithmic_bytes(M, N, K_BITS, act="sbvr", l=L_BITS)


def convert_bytes(N):
    return 2 * N + N * L_BITS // 8 + 4 * (N // G)


# ------------------------------------------------------------------ CPU oracle baseline
def cpu_baseline(budget_s: float = 15.0):
    import oracle
    shapes = layer_shapes()
    encs = []
    for idx, (name, M, N) in enumerate(shapes):
        pc, s16, b16, ri = synthetic.random_encoded(M, N, K_BITS, N_RATIO, seed=400 + idx)
        encs.append(oracle.Encoded(M, N, oracle.OracleConfig(K=K_BITS, n_ratio=N_RATIO), pc, s16, b16, ri, None))
    xs = [synthetic.activation(n, seed=900 + i)[0] for i, n in enumerate(INPUT_N)]
    # bounded sample: every 8th row of every matrix (same shapes and data), repeated within the budget
    stride = 8
    t0 = time.perf_counter()
    done_bytes, passes = 0, 0
    while True:
        xdec = []
        for x in xs:
            z, xp, sc = oracle.encode_vector(x, G, L_BITS)
            xdec.append(oracle.x_dec_sbvr(z, sc))
        for idx, (name, M, N) in enumerate(shapes):
            rows = np.arange(0, M, stride, dtype=np.int32)
            oracle.gemv_rows(encs[idx], xdec[INPUT_OF[name]], rows)
            done_bytes += len(rows) * (N * K_BITS // 8 + 5 * (N // G) + 4) + (N * L_BITS // 8 + 4 * (N // G))
        passes += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    c1 = oracle_c1_timing()
    return {"c1": c1, "value": done_bytes / dt / 1e9, "unit": "GB/s", "cores": oracle.max_threads(), "kind": "oracle",
            "sample": f"Llama-3-8B layer set, every {stride}th output row of each of the 7 projections "
                      f"(decode-then-dot fp64 O-Y + O-X activation conversion), {passes} passes in {dt:.1f}s",
            "seconds": dt}


def oracle_c1_timing():
    """SURVEY §8d.7 / BASELINE configs[0] (C1: 1024x1024 fp32 N(0,1), K=4, G=128, one x): the oracle's encode
    and GEMV wall time on all host cores and on one core.  Encode is timed on a bounded sample of rows (Algorithm
    1 costs ~tens of ms per group per core) and extrapolated to the 8192 groups of C1 (stated); the GEMV runs
    the full matrix."""
    import oracle
    W = synthetic.gaussian_weight(1024, 1024, seed=0, sigma=1.0)
    x = synthetic.activation(1024, seed=1)[0]
    cfg = oracle.OracleConfig(K=K_BITS)
    cores = oracle.max_threads()
    out = {"cores": cores, "cpu": _cpu_model(), "groups_total": 8192}
    for label, nth, rows in (("all_cores", cores, max(1, min(64, cores * 2))), ("1_core", 1, 1)):
        t0 = time.perf_counter()
        enc = oracle.encode_matrix(W[:rows], cfg, nthreads=nth)     # also sets the oracle's thread count
        dt = time.perf_counter() - t0
        gps = rows * 8 / dt
        z, xp, sc = oracle.encode_vector(x, G, L_BITS)
        full = oracle.Encoded(1024, 1024, cfg, np.tile(enc.planes[:1], (1024, 1, 1, 1)), np.tile(enc.s16[:1], (1024, 1)),
                              np.tile(enc.b16[:1], (1024, 1)), np.tile(enc.r_idx[:1], (1024, 1)), None)
        t1 = time.perf_counter()
        oracle.gemv_rows(full, oracle.x_dec_sbvr(z, sc))
        gdt = time.perf_counter() - t1
        out[label] = {"threads": nth, "encode_sample_groups": rows * 8, "encode_s_sample": round(dt, 3),
                      "encode_groups_per_s": round(gps, 2), "c1_encode_s_extrapolated": round(8192 / gps, 1),
                      "c1_gemv_s": round(gdt, 4)}
    oracle.encode_matrix(W[:1], cfg, nthreads=cores)               # restore the thread count
    return out


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ------------------------------------------------------------------ main SBVR arm
def run_sbvr(args, world, rank, local_rank, pg):
    import paper_2509_18172_b200 as sb
    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    cr = _Cudart()
    stream = torch.cuda.Stream(device)
    ring = args.ring
    with torch.cuda.stream(stream):
        layers = build_ring(sb, ring, world, rank, device)
        # the 4 layer inputs live in one buffer so a single sbvr_encode_vector launch converts all of them
        xcat = np.concatenate([synthetic.activation(n, seed=900 + i)[0] for i, n in enumerate(INPUT_N)])
        xs_host = [torch.from_numpy(xcat).pin_memory()]
        xs = [xs_host[0].to(device)]
        act_all = sb.encode_vector(xs[0])
        acts, g0 = [], 0
        for n in INPUT_N:
            ng = n // G
            acts.append(sb.SbvrActivation(sb.ACT_SBVR, n, 1, L_BITS, act_all.data[g0 * L_BITS * 4:(g0 + ng) * L_BITS * 4],
                                          act_all.scales[g0:g0 + ng]))
            g0 += ng
        if args.fused_conversion:                       # each GEMV converts its own input (Eq. 12 in its prologue)
            e0 = 0
            acts = []
            for n in INPUT_N:
                acts.append(sb.fp16q_activation(xs[0][e0:e0 + n], l=L_BITS))
                e0 += n
        # each ring layer's y's are views of one contiguous buffer (one device->host copy per step in e2e)
        yall = [torch.zeros(sum(r1 - r0 for (_, M, N, r0, r1, w, ws, xin) in mats), dtype=torch.float32, device=device)
                for mats in layers]
        ys = []
        for r, mats in enumerate(layers):
            off, views = 0, []
            for (_, M, N, r0, r1, w, ws, xin) in mats:
                views.append(yall[r][off:off + (r1 - r0)])
                off += r1 - r0
            ys.append(views)
        yfull = [torch.zeros(M, dtype=torch.float32, device=device) for (_, M, N, _, _) in FUSED]
        symm = symm_group = None
        if args.allgather == "symm" and args.step == "group":   # grouped launch with the all-gather in its epilogue
            symm_group = [sdist.SymmGroupRowShardedGemv([w for (_, M, N, r0, r1, w, ws, xin) in mats],
                                                        [M for (_, M, N, r0, r1, w, ws, xin) in mats], pg)
                          for mats in layers]
        elif args.allgather == "symm":                 # (at N = 1 too: exercises the same code path)
            symm = [[sdist.SymmRowShardedGemv(w, M, 1, pg, ws) for (_, M, N, r0, r1, w, ws, xin) in mats]
                    for mats in layers]
        y_host = [torch.zeros(M, dtype=torch.float32).pin_memory() for (_, M, N, _, _) in FUSED]
        # grouped step: the layer set's 4 GEMVs (independent problems over the converted inputs) in ONE persistent
        # sbvr_gemv_group launch; one workspace per ring layer
        group_probs = group_ws = None
        if args.step == "group":
            gacts = acts
            if args.xconv == "kernel":                 # the grouped kernel converts the fp16 inputs (Eq. 12) itself
                gacts, e0 = [], 0
                for n in INPUT_N:
                    gacts.append(sb.fp16q_activation(xs[0][e0:e0 + n], l=L_BITS))
                    e0 += n
            group_probs = [[(w, gacts[xin], ys[r][j]) for j, (name, M, N, r0, r1, w, ws, xin) in enumerate(layers[r])]
                           for r in range(ring)]
            group_ws = [sb.group_workspace(p) for p in group_probs]
    torch.cuda.synchronize()

    def step(r, events=None, span=None, e2e=False, xsrc=None):
        if e2e:
            for x, xh in zip(xs, xs_host):
                x.copy_(xh, non_blocking=True)
        if not args.fused_conversion and not (group_probs is not None and args.xconv == "kernel"):
            sb.encode_vector(xs[0] if xsrc is None else xsrc, out=act_all)
        if span is not None:
            cr.record_external(span[0], stream)
        if group_probs is not None:
            if events is not None:
                cr.record_external(events[0][0], stream)
            if symm_group is not None:
                symm_group[r]([p[1] for p in group_probs[r]])
            else:
                sb.gemv_group(group_probs[r], ws=group_ws[r])
            if events is not None:
                cr.record_external(events[0][1], stream)
            if world > 1 and symm_group is None:
                for j in range(len(layers[r])):
                    sdist.all_gather_rows_into(yfull[j], ys[r][j], group=pg)
        for j, (name, M, N, r0, r1, w, ws, xin) in enumerate(layers[r] if group_probs is None else []):
            if events is not None:
                cr.record_external(events[j][0], stream)
            if symm is not None:                        # all-gather fused into the GEMV epilogue (dist.py)
                symm[r][j](acts[xin])
            elif args.chain:                         # + L2 prefetch of the next GEMV's first units (next layer's qkv last)
                nxt = layers[r][j + 1][5] if j + 1 < len(layers[r]) else layers[(r + 1) % ring][0][5]
                sb.gemv_chain(w, acts[xin], nxt, y=ys[r][j], ws=ws)
            else:
                sb.gemv(w, acts[xin], y=ys[r][j], ws=ws)
            if events is not None:
                cr.record_external(events[j][1], stream)
            if world > 1 and symm is None:
                sdist.all_gather_rows_into(yfull[j], ys[r][j], group=pg)
        if span is not None:
            cr.record_external(span[1], stream)
        if e2e:
            for j in range(len(layers[r])):
                src = (symm[r][j].y_full[0] if symm is not None else symm_group[r].y_full[j] if symm_group is not None
                       else (yfull[j] if world > 1 else ys[r][j]))
                y_host[j].copy_(src, non_blocking=True)

    # --- capture graphs: one plain step graph per ring layer; span-instrumented copies (one event
    # pair around the 4 back-to-back GEMV launches, which stay chained by programmatic dependent
    # launch) replayed in one timed step out of EV_EVERY; per-GEMV-instrumented copies (events
    # between launches cut that chaining) replayed only after the timed region, as a breakdown.
    n_ev_graphs = 2
    # A decode step of a whole model is one CUDA graph: the timed graphs hold SPG consecutive steps (one
    # per ring layer, chained by programmatic dependent launch like the layers of a model); single-step graphs
    # serve a remainder of K that SPG does not divide.
    spg = max(1, min(args.steps_per_graph, args.steps))     # (a run of K < SPG steps is one K-step graph)
    ev_graphs, plain_graphs, split_graphs = [], [], []
    with torch.cuda.stream(stream):
        for _ in range(3):
            step(0)
        torch.cuda.synchronize()
        for r in range(ring):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step(r)
            plain_graphs.append(g)
        multi_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(multi_graph, stream=stream):
            for r in range(spg):
                step(r % ring)
        for gi in range(n_ev_graphs):
            span = (cr.event(), cr.event())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for r in range(spg):
                    step(r % ring, span=span if r == 1 % spg else None)
            ev_graphs.append((g, span, 0))
        for r in range(ring):
            evs = [(cr.event(), cr.event()) for _ in FUSED]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step(r, events=evs)
            split_graphs.append((g, evs))
        e2e_graphs = []
        for r in range(ring):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step(r, e2e=True)
            e2e_graphs.append(g)
        # e2e, pipelined as a serving loop would run it: every step's input is copied host -> device and its y
        # device -> host on a side stream, the next step's input while this step computes, this step's y while the
        # next one computes (per-step input buffers; one contiguous y per step).  Variants whose GEMVs read the fp16
        # input buffer directly (in-kernel conversion) or gather y across ranks keep the serial form below.
        e2e_pipelined = (world == 1 and symm is None and symm_group is None and not args.fused_conversion and
                         not (group_probs is not None and args.xconv == "kernel"))
        e2e_multi = torch.cuda.CUDAGraph()
        if e2e_pipelined:
            xh_e2e = [xs_host[0].clone().pin_memory() for _ in range(spg)]
            xd_e2e = [torch.empty_like(xs[0]) for _ in range(spg)]
            yh_e2e = [torch.zeros(yall[r % ring].numel(), dtype=torch.float32).pin_memory() for r in range(spg)]
            xd_e2e[0].copy_(xh_e2e[0])
            side = torch.cuda.Stream(device)
            evx = [torch.cuda.Event() for _ in range(spg)]
            evg = [torch.cuda.Event() for _ in range(spg)]
            torch.cuda.synchronize()
            with torch.cuda.graph(e2e_multi, stream=stream):
                side.wait_stream(stream)
                for r in range(spg):
                    if r > 0:
                        stream.wait_event(evx[r])
                    step(r % ring, xsrc=xd_e2e[r])
                    evg[r].record(stream)
                    with torch.cuda.stream(side):
                        nr = (r + 1) % spg                 # the next step's input (r = last: the next replay's first)
                        xd_e2e[nr].copy_(xh_e2e[nr], non_blocking=True)
                        evx[nr].record(side)
                        side.wait_event(evg[r])
                        yh_e2e[r].copy_(yall[r % ring], non_blocking=True)
                stream.wait_stream(side)
        else:
            with torch.cuda.graph(e2e_multi, stream=stream):
                for r in range(spg):
                    step(r % ring, e2e=True)
    torch.cuda.synchronize()

    # --- algorithmic bytes (whole job: full matrices, all ranks together)
    step_gemv_bytes = sum(gemv_bytes(sb, M, N) for (_, M, N, _, _) in FUSED)
    step_conv_bytes = sum(convert_bytes(n) for n in INPUT_N) * world
    step_bytes = step_gemv_bytes + step_conv_bytes
    rank_gemv_bytes = [gemv_bytes(sb, r1 - r0, N) for (_, M, N, r0, r1, w, ws, xin) in layers[0]]

    # Every replay below runs INSIDE `with torch.cuda.stream(stream)`: CUDAGraph.replay() launches on the
    # current stream, and the timing events are recorded on that same stream, so they bracket the GPU
    # work itself (round 1 replayed on the default stream while recording on `stream`, which timed only
    # the host's enqueue rate).
    with torch.cuda.stream(stream):
        # --- warmup + clock heat-up (untimed)
        for i in range(max(args.warmup, 3)):
            plain_graphs[i % ring].replay()
        torch.cuda.synchronize()
        sampler = ClockSampler(local_rank) if rank == 0 else None
        wall_heat = time.time()
        # (with N > 1 ranks every step graph holds an NCCL all-gather, so every rank must replay the same
        # number of steps: a fixed count, not a wall-clock deadline)
        if world > 1:
            for i in range(6000):
                plain_graphs[i % ring].replay()
                if i % 200 == 199:
                    torch.cuda.synchronize()
        else:
            heat_end = time.time() + 0.6
            i = 0
            while time.time() < heat_end:
                multi_graph.replay()
                i += 1
                if i % 200 == 0:
                    torch.cuda.synchronize()
        torch.cuda.synchronize()

        # --- timed region: exactly K steps (K // SPG multi-step graph replays + K % SPG single steps), barrier +
        # sync on both sides; an event after every replay
        n_multi, n_single = args.steps // spg, args.steps % spg
        span_ms, span_n = 0.0, 0
        # one replay in ev_every carries the span events (at most a quarter of them: the event nodes cut the
        # programmatic overlap around that step); a run too short for any gets one instrumented replay afterwards
        ev_every = min(EV_EVERY, max(4, n_multi // 4))
        pending = {}
        if world > 1:
            torch.distributed.barrier(group=pg)
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(n_multi + n_single + 1)]
        wall0 = time.time()
        evs[0].record(stream)
        for s in range(n_multi):
            if s % ev_every == ev_every - 1:
                gi = (s // ev_every) % n_ev_graphs
                if gi in pending:                  # read the previous replay of this graph before reusing its events
                    span_ms += cr.elapsed_ms(*ev_graphs[gi][1])
                    span_n += 1
                ev_graphs[gi][0].replay()
                pending[gi] = True
            else:
                multi_graph.replay()
            evs[s + 1].record(stream)
        for s in range(n_single):
            plain_graphs[s % ring].replay()
            evs[n_multi + s + 1].record(stream)
        torch.cuda.synchronize()
        wall1 = time.time()
        for gi in pending:
            span_ms += cr.elapsed_ms(*ev_graphs[gi][1])
            span_n += 1
        elapsed = evs[0].elapsed_time(evs[-1])
        if span_n == 0:                                 # (after the timed region: not part of `elapsed`)
            ev_graphs[0][0].replay()
            torch.cuda.synchronize()
            span_ms += cr.elapsed_ms(*ev_graphs[0][1])
            span_n += 1
        if world > 1:
            torch.distributed.barrier(group=pg)
        step_ms = ([evs[i].elapsed_time(evs[i + 1]) / spg for i in range(n_multi)] +
                   [evs[n_multi + i].elapsed_time(evs[n_multi + i + 1]) for i in range(n_single)])
        clocks = sampler.summary(wall_heat, wall1) if sampler else None
        if sampler:
            sampler.stop()

        # --- e2e: host (pinned) -> device inputs, kernels, device -> host outputs, every step
        e2e_steps = args.steps
        if world > 1:
            torch.distributed.barrier(group=pg)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(e2e_steps // spg):
            e2e_multi.replay()
        for s in range(e2e_steps % spg):
            e2e_graphs[s % ring].replay()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1)

    # --- max over ranks
    t = torch.tensor([elapsed, e2e_ms], dtype=torch.float64, device=device)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX, group=pg)
    elapsed, e2e_ms = float(t[0]), float(t[1])

    # per-GEMV breakdown (diagnostic, after the timed region): events between the launches
    per_gemv_ms = np.zeros(len(FUSED))
    n_split = 8 * ring
    with torch.cuda.stream(stream):
        for i in range(n_split):
            g, gevs = split_graphs[i % ring]
            g.replay()
            torch.cuda.synchronize()
            per_gemv_ms += [cr.elapsed_ms(a, b) if (group_probs is None or k == 0) else 0.0
                            for k, (a, b) in enumerate(gevs)]
    gemv_ms_avg = per_gemv_ms / n_split
    res = dict(elapsed=elapsed, e2e_ms=e2e_ms, step_bytes=step_bytes, step_gemv_bytes=step_gemv_bytes,
               gemv_ms_avg=gemv_ms_avg, rank_gemv_bytes=rank_gemv_bytes, clocks=clocks,
               span_ms_avg=span_ms / max(span_n, 1), span_n=span_n, step_ms=step_ms, ev_every=ev_every, spg=spg,
               wall_ms=(wall1 - wall0) * 1e3, e2e_pipelined=e2e_pipelined)
    h2d = sum(x.numel() * 2 for x in xs_host)
    d2h = sum(y.numel() * 4 for y in y_host)          # (= one step's contiguous y: the pipelined copy moves the same)
    res["h2d"], res["d2h"] = h2d, d2h
    return res, sb


def cublas_fp16_baseline(args, device, ring=2, steps=200):
    """torch.nn.functional.linear (cuBLAS) fp16 GEMV over the same layer set (dense fp16 weights)."""
    shapes = [(n, M, N, xin) for n, M, N, xin, _ in FUSED]
    g = torch.Generator(device="cpu").manual_seed(7)
    Ws = [[(torch.randn(M, N, generator=g, dtype=torch.float32) * 0.02).to(torch.float16).to(device)
           for (_, M, N, _) in shapes] for _ in range(ring)]
    xs = [torch.randn(n, dtype=torch.float16, device=device) for n in INPUT_N]
    outs = [torch.empty(M, dtype=torch.float16, device=device) for (_, M, N, _) in shapes]
    stream = torch.cuda.Stream(device)

    def step(r):
        for j, (name, M, N, xin) in enumerate(shapes):
            torch.matmul(Ws[r][j], xs[xin], out=outs[j])

    with torch.cuda.stream(stream):
        for _ in range(3):
            step(0)
        torch.cuda.synchronize()
        graphs = []
        for r in range(ring):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=stream):
                step(r)
            graphs.append(gr)
        spg = max(1, min(args.steps_per_graph, steps))
        multi = torch.cuda.CUDAGraph()                 # as the SBVR step: consecutive steps in one graph
        with torch.cuda.graph(multi, stream=stream):
            for r in range(spg):
                step(r % ring)
        for i in range(20):
            multi.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for s in range(steps // spg):
            multi.replay()
        b.record(stream)
        torch.cuda.synchronize()
    ms = a.elapsed_time(b) / (steps // spg * spg)
    byts = sum(2 * M * N + 2 * N + 2 * M for (_, M, N, _) in shapes)
    del Ws
    torch.cuda.empty_cache()
    return {"ms_per_step": ms, "GBps": byts / (ms * 1e-3) / 1e9, "bytes_per_step": byts,
            "how": "torch.matmul fp16 [M,N]x[N] (cuBLAS GEMV) on the same 4 fused matrices, one CUDA graph holding "
                   "the steps of a ring of 2 layers (470 MB > L2)"}


def _graph_stats(stream, launch, iters, replays=15):
    """Capture `iters` back-to-back launches (launch(i)) in one CUDA graph on `stream`, replay it `replays`
    times with CUDA events around each replay (on that stream), return per-launch microseconds:
    (median, p10, p90) over the replays."""
    with torch.cuda.stream(stream):
        for i in range(3):
            launch(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for i in range(iters):
                launch(i)
        g.replay()
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(replays + 1)]
        evs[0].record(stream)
        for r in range(replays):
            g.replay()
            evs[r + 1].record(stream)
        torch.cuda.synchronize()
    us = np.array([evs[r].elapsed_time(evs[r + 1]) * 1e3 / iters for r in range(replays)])
    return float(np.median(us)), float(np.percentile(us, 10)), float(np.percentile(us, 90))


def _ring_count(nbytes):
    return max(2, int(2.2 * 132e6 // max(nbytes, 1)) + 1)     # distinct copies: ring > 2.2x the 126 MB L2


def _cublas_us(device, M, N, T, iters=40):
    """fp16 dense GEMV / skinny GEMM on the same shape (torch.matmul -> cuBLAS), same ring/graph method."""
    stream = torch.cuda.Stream(device)
    g = torch.Generator(device="cpu").manual_seed(M + N)
    W0 = (torch.randn(M, N, generator=g) * 0.02).to(torch.float16).to(device)
    ring = _ring_count(2 * M * N)
    Ws = [W0] + [W0.clone() for _ in range(ring - 1)]
    x = torch.randn(N, T, dtype=torch.float16, device=device) if T > 1 else torch.randn(N, dtype=torch.float16, device=device)
    out = torch.empty((M, T) if T > 1 else (M,), dtype=torch.float16, device=device)
    med, p10, p90 = _graph_stats(stream, lambda i: torch.matmul(Ws[i % ring], x, out=out), iters)
    del Ws, W0
    torch.cuda.empty_cache()
    return med


def _record(sb, device, config, name, M, N, K, T, act_kind, algo, P=1, M_full=None, iters=60, cublas=True, seed=0):
    """One SURVEY §8d.8 result record: us/GEMV median/p10/p90 over graph replays of `iters` launches on a ring
    of distinct weight copies (> L2), algorithmic GB/s, fractions of 8 TB/s and of the measured copy peak,
    cuBLAS fp16 at the same shape and the speedup."""
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, N_RATIO, seed=seed + M + N + K)
    w0 = sb.pack_canonical(pc, s16, b16, ri, N_RATIO, device=device)
    ring = _ring_count(w0.nbytes)
    ws_ = [w0] + [sb.SbvrWeights(M, N, K, N_RATIO, w0.data.clone(), w0.ratio_pow.clone()) for _ in range(ring - 1)]
    wsp = [sb.Workspace.for_weights(w, T) for w in ws_]
    x = torch.from_numpy(synthetic.activation(N, seed=6, T=T)).to(device)
    act = sb.encode_vector(x) if act_kind == "sbvr" else sb.fp16_activation(x)
    y = torch.empty(T, M, dtype=torch.float32, device=device)
    stream = torch.cuda.Stream(device)
    med, p10, p90 = _graph_stats(stream, lambda i: sb.gemv_ex(ws_[i % ring], act, y=y, ws=wsp[i % ring], algo=algo), iters)
    byts = sb.algorithmic_bytes(M, N, K, act=act_kind, l=L_BITS, T=T)
    del ws_, wsp
    torch.cuda.empty_cache()
    peak, _ = measured_peak()
    gbps = byts / (med * 1e-6) / 1e9
    rec = {"config": config, "shape": name, "M": M, "N": N, "K": K, "l": L_BITS if act_kind == "sbvr" else None,
           "path": {"sbvr": "SBVR-x", "fp16": "fp16-x"}[act_kind] + "/" + {0: "auto", 1: "popc", 2: "tc", 3: "mma",
                                                                            4: "pipe", 5: "zt"}[algo],
           "T": T, "P": P, "bytes_alg": int(byts), "us_median": round(med, 3), "us_p10": round(p10, 3),
           "us_p90": round(p90, 3), "GBps": round(gbps, 1), "pct_8TBps": round(gbps / 80.0, 2),
           "pct_measured_peak": round(100 * gbps / peak, 2), "ring": ring}
    if M_full:
        rec["M_full"] = M_full
    if cublas:
        cu = _cublas_us(device, M, N, T)
        rec["cublas_us"] = round(cu, 3)
        rec["speedup_vs_cublas"] = round(cu / med, 3)
    return rec


def _group_record(sb, device, config, mats, P=1, iters=30, seed=0):
    """A SURVEY §8d.8-style record for one grouped launch (sbvr_gemv_group) over the matrices `mats` [(name, M, N)]
    (this rank's row shards at P ranks): us per launch median/p10/p90 over graph replays on a ring of distinct
    weight sets (> L2), algorithmic GB/s and fractions of 8 TB/s and of the measured copy peak."""
    sets, byts = [], 0
    base = []
    for j, (name, M, N) in enumerate(mats):
        pc, s16, b16, ri = synthetic.random_encoded(M, N, K_BITS, N_RATIO, seed=seed + 31 * j + M + N)
        base.append(sb.pack_canonical(pc, s16, b16, ri, N_RATIO, device=device))
        byts += sb.algorithmic_bytes(M, N, K_BITS, act="sbvr", l=L_BITS)
    ring = _ring_count(sum(w.nbytes for w in base))
    xs = [sb.encode_vector(torch.from_numpy(synthetic.activation(N, seed=60 + j)).to(device))
          for j, (_, M, N) in enumerate(mats)]
    ys = [torch.empty(M, dtype=torch.float32, device=device) for (_, M, N) in mats]
    for r in range(ring):
        ws_ = base if r == 0 else [sb.SbvrWeights(w.M, w.N, K_BITS, N_RATIO, w.data.clone(), w.ratio_pow.clone())
                                   for w in base]
        probs = [(w, x, y) for w, x, y in zip(ws_, xs, ys)]
        sets.append((probs, sb.group_workspace(probs)))
    stream = torch.cuda.Stream(device)
    med, p10, p90 = _graph_stats(stream, lambda i: sb.gemv_group(sets[i % ring][0], ws=sets[i % ring][1]), iters)
    del sets
    torch.cuda.empty_cache()
    peak, _ = measured_peak()
    gbps = byts / (med * 1e-6) / 1e9
    return {"config": config, "shape": "+".join(f"{n} {M}x{N}" for n, M, N in mats), "K": K_BITS, "l": L_BITS,
            "path": "SBVR-x/group", "T": 1, "P": P, "bytes_alg": int(byts), "us_median": round(med, 3),
            "us_p10": round(p10, 3), "us_p90": round(p90, 3), "GBps": round(gbps, 1), "pct_8TBps": round(gbps / 80.0, 2),
            "pct_measured_peak": round(100 * gbps / peak, 2), "ring": ring}


def _tensor_peak():
    """Measured dense bf16 TF/s (MEASURED_PEAKS.json, burst); fp16 runs at the bf16 rate (guide's nominal ratio 1)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"]), "measured (MEASURED_PEAKS.json bf16_tflops, burst; fp16 = bf16 rate)"
    except Exception:
        return 2250.0, "fallback (nominal 2.25 PFLOP/s dense fp16)"


def _prefill_record(sb, device, config, name, M, N, T, iters=20, seed=0):
    """f1 prefill (sbvr_prefill): us per call median/p10/p90 over graph replays on a ring of distinct weight
    copies (> L2), the weight stream's algorithmic GB/s (compressed bytes), the GEMM's TFLOP/s against the measured
    dense fp16 peak, cuBLAS fp16 GEMM at the same (M, N, T) and the speedup."""
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K_BITS, N_RATIO, seed=seed + M + N)
    w0 = sb.pack_canonical(pc, s16, b16, ri, N_RATIO, device=device)
    ring = _ring_count(w0.nbytes)
    ws_ = [w0] + [sb.SbvrWeights(M, N, K_BITS, N_RATIO, w0.data.clone(), w0.ratio_pow.clone()) for _ in range(ring - 1)]
    wsp = [sb.prefill_workspace(w, T) for w in ws_]
    X = torch.from_numpy(synthetic.activation(N, seed=7, T=T)).to(device)
    Y = torch.empty(T, M, dtype=torch.float32, device=device)
    stream = torch.cuda.Stream(device)
    med, p10, p90 = _graph_stats(stream, lambda i: sb.prefill(ws_[i % ring], X, Y, wsp[i % ring]), iters)
    wbytes = M * N * K_BITS // 8 + 5 * M * N // 128
    tflops = 2.0 * M * N * T / (med * 1e-6) / 1e12
    tpeak, _ = _tensor_peak()
    del ws_, wsp
    torch.cuda.empty_cache()
    cu = _cublas_us(device, M, N, T)
    return {"config": config, "shape": name, "M": M, "N": N, "K": K_BITS, "path": "prefill/fp16-decompress+tcgen05",
            "T": T, "us_median": round(med, 3), "us_p10": round(p10, 3), "us_p90": round(p90, 3),
            "weight_GBps": round(wbytes / (med * 1e-6) / 1e9, 1), "TFLOPs": round(tflops, 1),
            "frac_tensor_peak": round(tflops / tpeak, 4), "ring": ring, "cublas_us": round(cu, 3),
            "speedup_vs_cublas": round(cu / med, 3)}


def records(device):
    """one record per (config, shape, K, path, T, P) -- C2 Llama-3-8B decode set, C3 Llama-3-70B
    MLP row shards, C4 Qwen2.5-7B K sweep on both activation paths, C5 batched T = 1..64 -- plus f3."""
    import paper_2509_18172_b200 as sb
    out = []
    for name, M, N in synthetic.LLAMA3_8B_LAYER + [("qkv_fused", 6144, 4096), ("gate_up_fused", 28672, 4096)]:
        out.append(_record(sb, device, "C2 llama3_8b", name, M, N, K_BITS, 1, "sbvr", sb.ALGO_AUTO, iters=100))
    for name, M, N in synthetic.LLAMA3_70B_MLP[:2]:
        for P in (1, 2, 4, 8):
            out.append(_record(sb, device, "C3 llama3_70b_mlp_row_shard", name, M // P, N, K_BITS, 1, "sbvr",
                               sb.ALGO_AUTO, P=P, M_full=M, iters=40))
    # C3 per-rank MLP GEMVs as one grouped launch (fused gate_up + down row shards), P = 1/2/4/8 on one GPU
    for P in (1, 2, 4, 8):
        out.append(_group_record(sb, device, "C3 llama3_70b_mlp_row_shard_grouped",
                                 [("gate_up_proj", 57344 // P, 8192), ("down_proj", 8192 // P, 28672)], P=P,
                                 iters=20 if P <= 2 else 40))
    # C2 layer set as one grouped launch (the bench step's GEMV part, one launch per graph node)
    out.append(_group_record(sb, device, "C2 llama3_8b_grouped", [(n, M, N) for n, M, N, _, _ in FUSED], iters=40))
    for name, M, N in (("q_proj", 3584, 3584), ("k_proj", 512, 3584), ("gate_proj", 18944, 3584), ("down_proj", 3584, 18944)):
        for K in (2, 3, 4):
            for kind in ("sbvr", "fp16"):
                out.append(_record(sb, device, "C4 qwen25_7b", name, M, N, K, 1, kind, sb.ALGO_AUTO,
                                   cublas=(K == 4 and kind == "sbvr")))
    # C6 f1 prefill (FP16 decompression + tcgen05 GEMM) on the Llama-3-8B shapes
    for name, M, N in (("q_proj", 4096, 4096), ("gate_proj", 14336, 4096), ("down_proj", 4096, 14336)):
        for T in (16, 64, 256):
            out.append(_prefill_record(sb, device, "C6 llama3_8b_prefill", name, M, N, T))
    for name, M, N in (("q_proj", 4096, 4096), ("gate_proj", 14336, 4096)):
        for T in (1, 2, 4, 8, 16, 32, 64):
            out.append(_record(sb, device, "C5 llama3_8b_batched", name, M, N, K_BITS, T, "sbvr", sb.ALGO_AUTO,
                               iters=40 if T <= 16 else 20))
            if 2 <= T <= 16:
                for algo in (sb.ALGO_MMA, sb.ALGO_ZT):
                    out.append(_record(sb, device, "C5 llama3_8b_batched", name, M, N, K_BITS, T, "sbvr", algo,
                                       iters=40, cublas=False))
    return out


def sweeps(device):
    import paper_2509_18172_b200 as sb
    return {"records": records(device), "layer_chain_llama3_8b": layer_chain(sb, device)}


def layer_chain(sb, device, reps=20):
    """one synthetic Llama-3-8B decoder layer as deployed at batch 1 with every GEMV
    converting its own input (sbvr_encode_vector + sbvr_gemv for q, k, v, o, gate, up, down -- unfused,
    7 + 7 launches), one CUDA graph over a ring of layers (> L2), device time per layer (the TPOT-like
    per-layer GEMV latency of Table 3's setting).  Also the fused form (qkv and gate_up stacked,
    4 conversions) for comparison, and both with the conversion done in each GEMV's prologue (SBVR_ACT_FP16_Q:
    7 / 4 launches, bit-identical y)."""
    out = {}
    unf = [(n, M, N) for n, M, N in synthetic.LLAMA3_8B_LAYER]
    fus = [(n, M, N) for n, M, N, _, _ in FUSED]
    for label, mats, xq in (("unfused_7", unf, False), ("fused_4", fus, False),
                            ("unfused_7_in_kernel_conversion", unf, True), ("fused_4_in_kernel_conversion", fus, True)):
        ring = 3
        layers = []
        for r in range(ring):
            ws_ = []
            for i, (n, M, N) in enumerate(mats):
                pc, s16, b16, ri = synthetic.random_encoded(M, N, K_BITS, N_RATIO, seed=900 + 13 * r + i)
                w = sb.pack_canonical(pc, s16, b16, ri, N_RATIO, device=device)
                ws_.append((w, sb.Workspace.for_weights(w, 1), torch.empty(M, device=device),
                            torch.from_numpy(synthetic.activation(N, seed=i)).to(device)))
            layers.append(ws_)
        acts = [[sb.fp16q_activation(x[0]) if xq else sb.encode_vector(x) for (_, _, _, x) in L] for L in layers]
        stream = torch.cuda.Stream(device)
        with torch.cuda.stream(stream):
            def one(r):
                for (w, wsp, y, x), a in zip(layers[r], acts[r]):
                    if not xq:
                        sb.encode_vector(x, out=a)
                    sb.gemv(w, a, y=y, ws=wsp)
            for r in range(ring):
                one(r)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for i in range(reps):
                    one(i % ring)
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / reps
        byts = sum(sb.algorithmic_bytes(M, N, K_BITS, act="sbvr", l=L_BITS, T=1) for (_, M, N) in mats)
        out[label] = {"us_per_layer": round(us, 2), "launches_per_layer": (1 if xq else 2) * len(mats),
                      "GBps": round(byts / (us * 1e-6) / 1e9, 1),
                      "x32_layers_ms": round(32 * us / 1e3, 3)}
        del layers, acts
        torch.cuda.empty_cache()
    # unfused weights, launched by dependency level with the grouped kernel: (q, k, v) -> o -> (gate, up) -> down,
    # each level's inputs converted by one sbvr_encode_vector (q/k/v share x, gate/up share x): 4 + 4 launches,
    # the fused form's launch count without stacking the weights
    levels = [[0, 1, 2], [3], [4, 5], [6]]
    ring = 3
    layers = []
    for r in range(ring):
        ws_ = []
        for i, (n, M, N) in enumerate(unf):
            pc, s16, b16, ri = synthetic.random_encoded(M, N, K_BITS, N_RATIO, seed=900 + 13 * r + i)
            ws_.append((sb.pack_canonical(pc, s16, b16, ri, N_RATIO, device=device), torch.empty(M, device=device)))
        layers.append(ws_)
    xs = [torch.from_numpy(synthetic.activation(unf[lv[0]][2], seed=lv[0])).to(device) for lv in levels]
    acts = [sb.encode_vector(x) for x in xs]
    probs = [[[(layers[r][i][0], acts[li], layers[r][i][1]) for i in lv] for li, lv in enumerate(levels)]
             for r in range(ring)]
    gws = [[sb.group_workspace(pl) for pl in probs[r]] for r in range(ring)]
    stream = torch.cuda.Stream(device)
    with torch.cuda.stream(stream):
        def one_g(r):
            for li in range(len(levels)):
                sb.encode_vector(xs[li], out=acts[li])
                sb.gemv_group(probs[r][li], ws=gws[r][li])
        for r in range(ring):
            one_g(r)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for i in range(reps):
                one_g(i % ring)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.replay()
        b.record(stream)
        torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    byts = sum(sb.algorithmic_bytes(M, N, K_BITS, act="sbvr", l=L_BITS, T=1) for (_, M, N) in unf)
    out["unfused_7_grouped_by_level"] = {"us_per_layer": round(us, 2), "launches_per_layer": 8,
                                         "GBps": round(byts / (us * 1e-6) / 1e9, 1), "x32_layers_ms": round(32 * us / 1e3, 3)}
    del layers, acts, probs, gws
    torch.cuda.empty_cache()
    return out


def hadamard_throughput(device):
    """f4: randomized 128-block Hadamard rotation -- GB/s (read + write) rotating the fp32 Llama-3-8B
    down_proj weight (offline, before encoding) and the step's 4 fp16 activations (online), plus its
    effect on the encoder's mean group MSE for Student-t(3) weights (rotated-domain MSE = original-domain
    MSE: the rotation is orthogonal)."""
    import paper_2509_18172_b200 as sb
    out = {}
    for name, rows, N, dt in (("down_proj_weight_fp32", 4096, 14336, torch.float32),
                              ("step_activations_fp16", 4, 14336, torch.float16)):
        X = torch.randn(rows, N, device=device).to(dt)
        sg = torch.from_numpy(synthetic.hadamard_signs(N, seed=5)).to(device)
        Y = torch.empty_like(X)
        it = 20 if rows > 4 else 200
        st = torch.cuda.Stream(device)
        with torch.cuda.stream(st):
            sb.hadamard_rows(X, sg, 128, out=Y)
            g = torch.cuda.CUDAGraph()                   # launch-bound at the activation size: graph it
            with torch.cuda.graph(g, stream=st):
                for _ in range(it):
                    sb.hadamard_rows(X, sg, 128, out=Y)
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            g.replay()
            b.record(st)
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / it
        by = 2 * X.numel() * X.element_size()
        out[name] = {"rows": rows, "N": N, "block": 128, "us": round(us, 3), "GBps": round(by / us / 1e3, 1)}
    W = torch.from_numpy(synthetic.student_t_weight(512, 4096, seed=77)).to(device)
    sg = torch.from_numpy(synthetic.hadamard_signs(4096, seed=78)).to(device)
    _, m0 = sb.encode_weights(W, K=K_BITS, return_mse=True)
    _, m1 = sb.encode_weights(sb.hadamard_rows(W, sg, 128), K=K_BITS, return_mse=True)
    out["student_t3_512x4096_mean_group_mse"] = {"plain": m0.mean().item(), "rotated_b128": m1.mean().item()}
    return out


def encode_throughput(device):
    """Strict fp64 GPU encoder throughput on one Llama-3-8B q_proj (4096x4096, sigma 0.02): groups/s."""
    import paper_2509_18172_b200 as sb
    W = torch.from_numpy(synthetic.gaussian_weight(4096, 4096, seed=401, sigma=0.02)).to(device)
    sb.encode_weights(W[:256].contiguous(), K=K_BITS)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _, m_full_all = sb.encode_weights(W, K=K_BITS, return_mse=True)
    b.record()
    torch.cuda.synchronize()
    s = a.elapsed_time(b) / 1e3
    # f2 storage (reading A23): coefficient table (256 entries) + a 1-byte index per group
    a.record()
    w_idx, m_idx = sb.encode_weights_indexed(W, K=K_BITS, n_table=256)
    b.record()
    torch.cuda.synchronize()
    s_idx = a.elapsed_time(b) / 1e3
    indexed = {"n_table": 256, "table_entries": int(w_idx.coef_table[0].item()), "seconds": round(s_idx, 3),
               "groups_per_s": round(4096 * 4096 / G / s_idx), "meta_bytes_per_group": 1.0,
               "weight_bytes": int(w_idx.data.numel()), "weight_bytes_5B_meta": int(sb.weights_bytes(4096, 4096, K_BITS)[0]),
               "mean_mse": m_idx.mean().item(), "mean_mse_full_search": m_full_all.mean().item(),
               "max_mse": m_idx.max().item(), "max_mse_full_search": m_full_all.max().item()}
    del w_idx, m_idx
    groups = 4096 * 4096 // G
    # C5 (ii): the whole Llama-3-8B layer set (7 matrices, 218 M params, 1.70 M groups) encoded back to back
    t_layer, g_layer = 0.0, 0
    for i, (name, M, N) in enumerate(synthetic.LLAMA3_8B_LAYER):
        Wl = torch.from_numpy(synthetic.gaussian_weight(M, N, seed=402 + i, sigma=0.02)).to(device)
        torch.cuda.synchronize()
        a.record()
        sb.encode_weights(Wl, K=K_BITS)
        b.record()
        torch.cuda.synchronize()
        t_layer += a.elapsed_time(b) / 1e3
        g_layer += M * N // G
        del Wl
    layer = {"matrices": 7, "groups": g_layer, "params": g_layer * G, "seconds": round(t_layer, 3),
             "groups_per_s": round(g_layer / t_layer), "params_per_s": round(g_layer * G / t_layer),
             "full_model_32_layers_s_extrapolated": round(32 * t_layer, 1)}
    out = {"layer_set_llama3_8b": layer, "indexed": indexed,
           "shape": "4096x4096", "seconds": s, "groups_per_s": groups / s, "params_per_s": groups * G / s,
           "search_space": "16x64x16 (R x S x B), strict fp64",
           "full_llama3_8b_extrapolated_s": 54525952 / (groups / s)}
    # fast mode (strict = 0): fp32 scan + fp64 re-evaluation of the near-best entries
    a.record()
    w_fast, m_fast = sb.encode_weights(W, K=K_BITS, return_mse=True, strict=False)
    b.record()
    torch.cuda.synchronize()
    sf = a.elapsed_time(b) / 1e3
    w_strict = sb.encode_weights(W, K=K_BITS)
    torch.cuda.synchronize()
    out["fast"] = {"seconds": round(sf, 3), "groups_per_s": round(groups / sf), "speedup_vs_strict": round(s / sf, 2),
                   "identical_to_strict": bool(torch.equal(w_fast.data, w_strict.data)),
                   "mean_mse": m_fast.mean().item(), "mean_mse_strict": m_full_all.mean().item(),
                   "full_llama3_8b_extrapolated_s": round(54525952 / (groups / sf), 1)}
    del w_fast, w_strict
    # f2: the encode-time coefficient cache (per-row MRU cache of 8, moving-average admission)
    _, m_full = sb.encode_weights(W[:512].contiguous(), K=K_BITS, return_mse=True)
    a.record()
    _, m_c, hit = sb.encode_weights_cached(W, K=K_BITS, cache_size=8, ema_alpha=0.1)
    b.record()
    torch.cuda.synchronize()
    sc = a.elapsed_time(b) / 1e3
    out["cached"] = {"cache_size": 8, "ema_alpha": 0.1, "seconds": sc, "groups_per_s": groups / sc,
                     "speedup_vs_full_search": s / sc, "hit_rate": hit.float().mean().item(),
                     "mean_mse_cached": m_c.mean().item(),
                     "mean_mse_full_first512rows": m_full.mean().item(),
                     "mean_mse_cached_first512rows": m_c[:512].mean().item()}
    return out


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ncu dram bytes per launch of the step's GEMV launches (tools/traffic_from_ncu.py)
TRAFFIC_FILE = {"chain": "r02_ncu_traffic.json", "group": "r02_ncu_traffic_group.json"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="sbvr", choices=["sbvr", "reference"])
    ap.add_argument("--ring", type=int, default=4)
    ap.add_argument("--steps-per-graph", type=int, default=32,
                    help="consecutive steps per timed CUDA graph: Llama-3-8B's 32 decoder layers form one decode graph "
                         "(P:447); the layers cycle through the --ring distinct weight sets")
    ap.add_argument("--fused-conversion", action="store_true",
                    help="no sbvr_encode_vector launch: every GEMV converts its fp16 input in its prologue "
                         "(SBVR_ACT_FP16_Q, bit-identical)")
    ap.add_argument("--chain", action="store_true",
                    help="launch the step's GEMVs with sbvr_gemv_chain (L2 prefetch of the next GEMV's first units; "
                         "measured no gain: profiles/r02_chain_ab.txt)")
    ap.add_argument("--step", default="group", choices=["group", "chain"],
                    help="group: the layer set's 4 GEMVs in one persistent sbvr_gemv_group launch (default); chain: "
                         "4 sbvr_gemv launches chained by programmatic dependent launch")
    ap.add_argument("--xconv", default="launch", choices=["kernel", "launch"],
                    help="group step: one sbvr_encode_vector launch precedes the grouped GEMV (default), or the grouped kernel converts the fp16 layer inputs itself (Eq. 12, bit-identical; "
                         "measured ~3.5 us slower per step: the first read of the freshly converted planes is slow)")
    ap.add_argument("--allgather", default="nccl", choices=["nccl", "symm"],
                    help="N > 1: join y with an NCCL all-gather, or store it to every rank from the GEMV epilogue "
                         "(symmetric memory, dist.SymmRowShardedGemv)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--no-encode", action="store_true")
    ap.add_argument("--no-sweeps", action="store_true")
    args = ap.parse_args()
    if args.fused_conversion or args.chain:
        args.step = "chain"                        # those variants exist on the per-GEMV launches only

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    pg = None

    if args.impl == "reference":
        return run_reference(args, world, rank)

    if world > 1 or args.allgather == "symm":
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        torch.distributed.init_process_group("nccl", rank=rank, world_size=world,
                                             device_id=torch.device("cuda", local_rank))
        pg = torch.distributed.group.WORLD
    res, sb = run_sbvr(args, world, rank, local_rank, pg)
    device = torch.device("cuda", local_rank)
    extra = {}
    if rank == 0:
        if not args.no_cublas:
            try:
                extra["cublas"] = cublas_fp16_baseline(args, device)
            except Exception as e:  # pragma: no cover
                extra["cublas"] = {"error": str(e)}
        if not args.no_encode:
            try:
                extra["encode"] = encode_throughput(device)
                extra["hadamard"] = hadamard_throughput(device)
            except Exception as e:  # pragma: no cover
                extra["encode"] = {"error": str(e)}
        if not args.no_sweeps and world == 1:
            try:
                extra["sweeps"] = sweeps(device)
            except Exception as e:  # pragma: no cover
                extra["sweeps"] = {"error": str(e)}
        if not args.no_cpu_baseline and world == 1:
            extra["cpu"] = cpu_baseline()
    if world > 1:
        torch.distributed.barrier(group=pg)
    if rank != 0:
        torch.distributed.destroy_process_group()
        return

    K, W = args.steps, args.warmup
    ms_per_step = res["elapsed"] / K
    value = res["step_bytes"] / (ms_per_step * 1e-3) / 1e9
    peak, peak_src = measured_peak()
    gemv_ms = res["gemv_ms_avg"]
    shapes = layer_shapes()
    per = []
    group = args.step == "group"
    for j, (name, M, N, xin, members) in enumerate(FUSED if not group else []):
        b = res["rank_gemv_bytes"][j]
        per.append({"gemv": name, "projections": list(members), "M": M, "N": N, "rows_per_rank": M // world,
                    "us_serialized": round(gemv_ms[j] * 1e3, 3), "GBps": round(b / (gemv_ms[j] * 1e-3) / 1e9, 1)})
    if group:
        b = sum(res["rank_gemv_bytes"])
        per.append({"gemv": "group(" + ",".join(f[0] for f in FUSED) + ")", "us_serialized": round(gemv_ms[0] * 1e3, 3),
                    "GBps": round(b / (gemv_ms[0] * 1e-3) / 1e9, 1)})
    n_launch_gemv = 1 if group else len(FUSED)
    tot_b = sum(res["rank_gemv_bytes"])
    achieved = tot_b / (res["span_ms_avg"] * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", TRAFFIC_FILE[args.step])
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("traffic_bytes_per_launch_mean")
        except Exception:
            traffic = None
    e2e_val = res["step_bytes"] / (res["e2e_ms"] / K * 1e-3) / 1e9
    conv_launch = 0 if (args.fused_conversion or (group and args.xconv == "kernel")) else 1
    launches = K * (conv_launch + n_launch_gemv)
    sm = np.asarray(res["step_ms"]) * 1e3
    step_stats = {"us_median": round(float(np.median(sm)), 3), "us_p10": round(float(np.percentile(sm, 10)), 3),
                  "us_p90": round(float(np.percentile(sm, 90)), 3), "us_mean": round(float(sm.mean()), 3)}
    # self-consistency of the headline (a number that fails one of these is not a measurement):
    #  (1) the events bracket the GPU work: the device time of the K steps is not much shorter than the host's wall
    #      time from the first event record to the synchronize after the last replay (replays are enqueued far
    #      faster than they run; round 1's events on an idle stream measured ~1/10 of the wall time);
    #  (2) the step cannot move its algorithmic bytes faster than the HBM peak (+5 % for run-to-run);
    #  (3) the end-to-end step (plus host<->device copies) cannot be shorter than the device-resident one.
    wall_ms = res["wall_ms"]
    checks = {"device_ms_ge_0.8_wall_ms": [round(res["elapsed"], 3), round(wall_ms, 3)],
              "value_le_1.05_peak": [round(value, 1), round(1.05 * peak * world, 1)],
              "e2e_step_ge_step_us": [round(res["e2e_ms"] / K * 1e3, 3), round(ms_per_step * 1e3, 3)]}
    # (the wall-time check needs a steady state: it is skipped below 20 ms of wall time, where Python's replay loop
    # and a profiler's serialisation dominate)
    ok = ((res["elapsed"] >= 0.8 * wall_ms or wall_ms < 20.0) and value <= 1.05 * peak * world
          and res["e2e_ms"] / K >= 0.99 * ms_per_step)
    if not ok:
        raise SystemExit(f"bench self-check failed (timing does not bracket the GPU work): {checks}")
    out = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic: random SBVR-encoded weights (uniform bit-planes, fp16 scale/bias, uniform ratio index; "
                "kernel time is data-independent), x ~ N(0,1) fp16",
        "config": {"workload": "llama3_8b_decode_layer_set_w4a8",
                   "projections": [f"{n} {M}x{N}" for n, M, N in shapes],
                   "gemvs_per_step": [f"{n} {M}x{N} = {'+'.join(m)}" for n, M, N, _, m in FUSED],
                   "K": K_BITS, "l": L_BITS, "group": G, "batch": 1, "ring_layers": args.ring,
                   "steps_per_graph": args.steps_per_graph,
                   "l2": "inputs larger than L2: ring of 4 distinct layer weight sets (468 MB) cycled every step",
                   "parallelism": f"row-sharded over {world} GPU(s)" + ((" + NCCL all-gather of y" if args.allgather == "nccl" else
                                                                       " + y stored to every rank by the GEMV epilogue "
                                                                       "(symmetric memory) + signal-pad barrier")
                                                                      if world > 1 else ""),
                   "path": (("sbvr_encode_vector x1 (the 4 layer inputs) + " if args.xconv == "launch" else "") +
                            "sbvr_gemv_group x1 over the layer set (fused qkv, o, fused gate_up, down as 4 independent "
                            "problems of one persistent launch" + ("" if args.xconv == "launch" else ", whose prologue "
                            "converts the 4 fp16 inputs to SBVR-x, Eq. 12") + "; bit-sliced "
                            "AND/popcount on the int8 tensor pipe, mma.sync m16n8k32 u8, kernel gemv_group), "
                            f"{args.steps_per_graph} steps (decoder layers) per CUDA graph, programmatic dependent "
                            "launch" if group else
                            "sbvr_encode_vector x1 (the 4 layer inputs) + sbvr_gemv x4 (fused qkv, o, fused gate_up, "
                            "down; bit-sliced AND/popcount on the int8 tensor pipe, mma.sync m16n8k32 u8, kernel "
                            f"gemv_mma), {args.steps_per_graph} steps (decoder layers) per CUDA graph, programmatic "
                            "dependent launch"),
                   "step": args.step, "x_conversion": ("in the GEMV kernel" if (args.fused_conversion or (
                       group and args.xconv == "kernel")) else "sbvr_encode_vector launch")},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                     "kernel": ("gemv_group_kernel<4> (the step's one grouped GEMV launch)" if group else
                                "gemv_mma_kernel<4,4,1,false,false,false,false,false> (the 4 GEMV launches of a step)"),
                     "how": "algorithmic bytes per launch / average launch duration over the step's GEMV launches "
                            "(= their summed bytes / the CUDA-event span around them; external event nodes in "
                            f"one step of {res['span_n']} of the {K // res['spg']} timed {res['spg']}-step graph replays, every "
                            f"{res['ev_every']}th); traffic = ncu dram "
                            "read+write bytes per launch (profiles/" + TRAFFIC_FILE[args.step] + ")",
                     "gemv_span_us": round(res["span_ms_avg"] * 1e3, 3),
                     "algorithmic_bytes_per_launch": round(tot_b / n_launch_gemv),
                     # (the event nodes around the measured launches cut their programmatic overlap with the
                     # neighbouring launches, so `achieved` is conservative; the same bytes over the steady-state step)
                     "achieved_steady_state": round(tot_b / (ms_per_step * 1e-3) / 1e9, 1),
                     "frac_steady_state": round(tot_b / (ms_per_step * 1e-3) / 1e9 / peak, 4)},
        "per_gemv": per,
        "per_gemv_how": "diagnostic after the timed region: event nodes between the 4 launches (no launch "
                        "overlap), so each figure includes a full launch + ramp",
        "pct_of_8TBps": round(achieved / 8000 * 100, 2),
        "e2e": {"value": round(e2e_val, 1), "unit": "GB/s", "h2d_bytes_per_step": res["h2d"],
                "d2h_bytes_per_step": res["d2h"], "ms_per_step": round(res["e2e_ms"] / K, 5),
                "how": ("every step: its fp16 inputs pinned host -> device and its y device -> host, on a side stream "
                        "overlapped with the neighbouring steps' compute (per-step input buffers), inside the same "
                        f"{res['spg']}-step graphs" if res["e2e_pipelined"] else
                        "every step: inputs host -> device, compute, y device -> host, serialised on one stream")},
        "gpu_launches": launches,
        "clocks": res["clocks"],
        "step_us": step_stats,
        "self_check": {"ok": True, **checks},
        "timing": f"K steps = K // {res['spg']} replays of a CUDA graph holding {res['spg']} consecutive steps (the "
                  f"decoder layers of one Llama-3-8B decode graph, cycling through {args.ring} distinct weight sets > L2, "
                  "chained by programmatic dependent launch) + K % "
                  f"{res['spg']} single-step graphs; CUDA events on the replay stream after every replay (each replay and "
                  "event runs under torch.cuda.stream(stream)); value = step algorithmic bytes x K / (last event - "
                  "first event); step_us = replay time / steps in it; barrier + synchronize on both sides; max over "
                  "ranks",
    }
    if "cublas" in extra:
        cb = extra["cublas"]
        out["vs_cublas_fp16"] = dict(cb)
        if "ms_per_step" in cb:
            out["vs_cublas_fp16"]["speedup_step"] = round(cb["ms_per_step"] / ms_per_step, 3)
            out["vs_cublas_fp16"]["speedup_gemv_only"] = round(cb["ms_per_step"] / res["span_ms_avg"], 3)
    if "encode" in extra:
        out["encode"] = extra["encode"]
    if "hadamard" in extra:
        out["hadamard"] = extra["hadamard"]
    if "sweeps" in extra:
        out["sweeps"] = extra["sweeps"]
    if "cpu" in extra:
        out["cpu_baseline"] = extra["cpu"]
    print(json.dumps(out), flush=True)


def run_reference(args, world, rank):
    """Reference arm = the CPU oracle as it stands, on this workload's metric/unit (rank 0 only)."""
    if world > 1 and rank != 0:
        return
    import oracle
    oracle.build()
    shapes = layer_shapes()
    encs = []
    for idx, (name, M, N) in enumerate(shapes):
        pc, s16, b16, ri = synthetic.random_encoded(M, N, K_BITS, N_RATIO, seed=400 + idx)
        encs.append(oracle.Encoded(M, N, oracle.OracleConfig(K=K_BITS, n_ratio=N_RATIO), pc, s16, b16, ri, None))
    xs = [synthetic.activation(n, seed=900 + i)[0] for i, n in enumerate(INPUT_N)]

    def one_step(stride):
        xdec = []
        for x in xs:
            z, xp, sc = oracle.encode_vector(x, G, L_BITS)
            xdec.append(oracle.x_dec_sbvr(z, sc))
        nbytes = 0
        for idx, (name, M, N) in enumerate(shapes):
            rows = np.arange(0, M, stride, dtype=np.int32)
            oracle.gemv_rows(encs[idx], xdec[INPUT_OF[name]], rows)
            nbytes += len(rows) * (N * K_BITS // 8 + 5 * (N // G) + 4)
        nbytes += sum(n * L_BITS // 8 + 4 * (n // G) + 2 * n for n in INPUT_N)
        return nbytes

    # size the per-step sample so that warmup + K steps take about 90 s of host time
    t0 = time.perf_counter()
    one_step(64)
    t64 = time.perf_counter() - t0
    target = 90.0 / max(args.steps + args.warmup, 1)
    stride = 64
    while stride > 1 and t64 * 64 / (stride // 2) <= target:
        stride //= 2
    while stride < 4096 and t64 * 64 / stride > target:
        stride *= 2
    for _ in range(max(args.warmup, 1)):
        one_step(stride)
    steps = args.steps
    t0 = time.perf_counter()
    tot = 0
    for _ in range(steps):
        tot += one_step(stride)
    dt = time.perf_counter() - t0
    val = tot / dt / 1e9
    out = {"impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "GB/s", "n_gpus": world,
           "steps": steps, "warmup": args.warmup, "ms_per_step": round(dt / steps * 1e3, 3), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (same seeds as the SBVR arm)",
           "config": {"workload": "llama3_8b_decode_layer_set_w4a8", "sample": f"every {stride}th output row"},
           "cpu_baseline": {"value": round(val, 3), "unit": "GB/s", "cores": oracle.max_threads(), "kind": "oracle",
                            "sample": f"every {stride}th output row of the 7 projections, decode-then-dot fp64"},
           "e2e": {"value": round(val, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
