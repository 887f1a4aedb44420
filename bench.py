"""pi0 inference latency on B200 — the BASELINE.json headline metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--views V --prompt P]

Workload (BASELINE.json configs[1], the paper headline): pi0 with 2 views of 224x224
(512 image tokens), empty prompt, chunk 63, 10 flow steps, random-init weights
(rtvla::gen_weights seed 1, on device) and synthetic inputs (rtvla::gen_inputs seed 1).

One "step" = one full inference (VE -> LLM prefill -> 10 AE flow steps -> Euler) = one replay of
the captured CUDA graph.  `value` = p50 latency over K device-timed replays (CUDA events on the
replay stream, inputs resident in HBM); `e2e` = p50 latency of the public API call
Engine.run(host fp64 inputs) -> host fp64 actions (H2D + replay + D2H inside the timed region).
Multi-GPU: one independent replica per GPU ("replicas only"): the metric is the
per-inference latency (max over ranks) and `throughput_inf_per_s` the aggregate rate.

`parity`: the benched engine's actions on the seed-1 inputs against the committed full-scale
golden of the same config (tests/golden/full_<cfg>.json, the reference's fp64 output): max-abs,
floored relative error and cosine (beside every GPU number).

Multi-GPU: `--gpus N` without torchrun re-launches itself under torch.distributed.run with N
ranks; under torchrun WORLD_SIZE must equal --gpus.  Ranks share nothing on the data path:
the only collectives are the gloo (CPU) barrier and max-reduce of the timings.

`--impl reference` times the reference's own CPU implementation: ONE full-scale
rtvla::evaluate (compiled unmodified from /root/reference into oracle/_ref, -O3 like the
reference's Release build) of the benched config on rank 0 -- graph build, gen_weights and
gen_inputs untimed, the evaluate call timed by the wall clock.  It is single-threaded (the
reference has no internal parallelism) and takes ~20-25 min at 2 views, so this arm always
reports steps = 1, warmup = 0 whatever --steps/--warmup say.
"""
from __future__ import annotations

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

METRIC = "p50 π0 inference latency (ms) at 1/2/3 views, chunk 63, 10 flow steps"


def reduce_over_ranks(values, op: str = "max"):
    """Max (or min) over ranks of per-rank numbers (the contract: every multi-GPU number is the
    max over ranks).  Over the gloo (CPU) group: replicas share no data-path collective, so no
    NCCL communicator is ever created.  No-op at world size 1."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(v) for v in values]
    t = torch.tensor([float(v) for v in values], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.MIN)
    return [float(v) for v in t.tolist()]


def init_replicas(gpus: int):
    """One process per GPU.  Under torchrun WORLD_SIZE must equal --gpus; the gloo group is
    only used for the barrier and the timing reduction (replicas only)."""
    ws, rank, local = _dist()
    if ws != gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={ws} but --gpus {gpus}")
    if ws > 1:
        import datetime

        import torch.distributed as dist
        # bounded: a rank that dies must not leave the others in a barrier for the default 30 min
        dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=600))
    return ws, rank, local


def spawn_replicas(argv, gpus: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch under torch.distributed.run, N ranks."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def _nccl_used() -> bool:
    import torch.distributed as dist
    return bool(dist.is_initialized() and dist.get_backend() == "nccl")


def staging_threads(ws: int) -> int:
    """Host helper threads per replica for the patch conversion (engine.cu stage_patches_bf16):
    3 on a dedicated host, fewer when N replicas share the cores."""
    if "PI0B_STAGING_THREADS" in os.environ:
        return int(os.environ["PI0B_STAGING_THREADS"])
    return max(0, min(3, (os.cpu_count() or 4) // max(ws, 1) - 1))


def golden_parity(cfg, y) -> dict | None:
    """Actions vs the committed full-scale golden of this config (reference fp64 output, seed 1)."""
    tag = f"{cfg.views}v" + (f"{cfg.prompt_tokens}p" if cfg.prompt_tokens else "")
    path = os.path.join(ROOT, "tests", "golden", f"full_{tag}.json")
    if not os.path.exists(path):
        return None
    ref = np.array(json.load(open(path))["actions"], dtype=np.float64).reshape(y.shape)
    d = y - ref
    floor = 0.1 * np.sqrt(np.mean(ref * ref))
    return {"golden": os.path.relpath(path, ROOT), "max_abs": float(np.abs(d).max()),
            "rms_err": float(np.sqrt(np.mean(d * d))), "rms_ref": float(np.sqrt(np.mean(ref * ref))),
            "rel": float(np.max(np.abs(d) / np.maximum(np.abs(ref), floor))),
            "cos": float((y.ravel() @ ref.ravel()) / (np.linalg.norm(y) * np.linalg.norm(ref)))}


def ve_shard_bench(cfg, ws: int, rank: int, local: int, steps: int, warmup: int, single_p50: float) -> dict | None:
    """SURVEY.md 8(e) / north_star: the view-sharded SigLIP stage at G = views GPUs (ranks < G):
    each rank encodes its own view(s) and the layers' q|k|v rows plus the final llm.proj_in rows
    are exchanged over NVLink peer memory (CUDA IPC mappings, the engine's fused push + release
    kernel, kernels_misc.cu); rank 0 runs the LLM and the action expert.  Latency = rank 0's
    device-timed full inference (CUDA events around its replay, the peers replaying their prefix
    at the same time after a host rendezvous).  Reported beside the single-GPU p50 so the
    "only where it lowers latency" question is answered by the measurement.  Every rank takes
    part in the same sequence of gloo collectives; any failure aborts the experiment on all ranks
    and is reported, never raised."""
    import torch.distributed as dist
    from paper_2510_26742_b200 import engine as E
    from paper_2510_26742_b200.inputs import gen_inputs
    G = cfg.views
    if ws < G or G < 2:
        return None
    part = rank < G
    eng, opened, err = None, [], None

    first_err = [None]  # the first failure reported by any rank (for rank 0's line)

    def agree(ok: bool) -> bool:
        flags = [None] * ws
        dist.all_gather_object(flags, (ok, err))
        for f_ok, f_err in flags:
            if not f_ok and first_err[0] is None:
                first_err[0] = f_err
        return all(f[0] for f in flags)

    try:
        if part:
            eng = E.Engine(cfg, device=local, ve_shards=G, ve_shard=rank)
            eng.gen_weights(1)
            mine = [E.ipc_export(p) for p in eng.ve_buffers().as_list()]
        else:
            mine = None
    except Exception as e:  # noqa: BLE001
        err, mine = f"rank {rank} setup: {e}"[:300], None
    handles = [None] * ws
    dist.all_gather_object(handles, mine)
    ok = err is None and all(h is not None for h in handles[:G])
    if part and ok:
        try:
            peers = []
            for g in range(G):
                if g == rank:
                    peers.append(eng.ve_buffers())
                else:
                    ptrs = [E.ipc_open(h) for h in handles[g]]
                    opened += ptrs
                    peers.append(E.VeBuffers.from_list(ptrs))
            eng.set_ve_peers(peers)
        except Exception as e:  # noqa: BLE001
            err, ok = f"rank {rank} peers: {e}"[:300], False
    if not agree(ok):
        res = {"gpus": G, "error": first_err[0] or err or "setup failed on another rank"}
    else:
        x = gen_inputs(cfg, 1)
        times, y, all_ok = [], None, True
        timer = DeviceTimer() if part else None
        for i in range(warmup + steps):
            all_ok = agree(ok)   # one collective per iteration on every rank: a failure anywhere stops all
            if not all_ok:
                break
            try:
                if rank == 0:
                    if y is None:   # first call: uploads the inputs and captures the graph
                        y = eng.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
                        continue
                    ms = timer.time(lambda st: eng.replay(0, st))
                    if i >= warmup:
                        times.append(ms)
                elif part:
                    if i == 0:
                        eng.run_prefix(x["patches"], x.get("prompt"))
                    else:
                        timer.time(lambda st: eng.replay(1, st))
            except Exception as e:  # noqa: BLE001
                err, ok = f"rank {rank} run: {e}"[:300], False
        all_ok = agree(ok) and all_ok
        if rank == 0 and all_ok and times:
            p50 = float(np.median(times))
            res = {"gpus": G, "p50_ms": round(p50, 4), "p90_ms": round(float(np.percentile(times, 90)), 4),
                   "steps": len(times), "single_gpu_p50_ms": round(single_p50, 4),
                   "lowers_latency": bool(p50 < single_p50), "parity": golden_parity(cfg, y),
                   "method": "rank 0 device-timed replay (CUDA events); peers replay their VE prefix after the same "
                             "gloo rendezvous; K/V rows + proj_in rows over CUDA-IPC peer memory"}
        else:
            res = {"gpus": G, "error": first_err[0] or err or "no timed steps"}
    for ptr in opened:
        try:
            E.ipc_close(ptr)
        except Exception:  # noqa: BLE001
            pass
    if eng is not None:
        eng.close()
    return res if rank == 0 else None


class DeviceTimer:
    """CUDA events around fn(stream handle) on a dedicated (non-legacy) stream; returns ms."""

    def __init__(self):
        import torch
        self._torch = torch
        self.stream = torch.cuda.Stream()

    def time(self, fn) -> float:
        t = self._torch
        a, b = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        a.record(self.stream)
        fn(self.stream.cuda_stream)
        b.record(self.stream)
        b.synchronize()
        return a.elapsed_time(b)


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: through NVML every 10 ms
    (pynvml, from nvidia_ml_py), else nvidia-smi every 0.2 s (each call takes ~0.3 s, so a short
    timed region gets one or two samples)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits, in the order of Q's four reason columns
    BITS = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal_slowdown, sw_thermal_slowdown, sw_power_cap

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.source = "nvidia-smi"
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self) -> bool:
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return False
        self.source = "nvml"
        while not self._stop.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                why = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(sm), str(mx), "0"] + ["Active" if why & b else "Not Active" for b in self.BITS])
            except Exception:
                pass
            self._stop.wait(0.01)
        return True

    def _run(self):
        if self._run_nvml():
            return
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 7:
                    self.rows.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": self.source}


def cpu_baseline_port(cfg, threads: int) -> dict:
    """The fp64 restatement (oracle/pi0_oracle.cpp, bitwise == reference) on a reduced-depth sample of
    the same workload (full widths and token counts, 1 VE layer, 2 LLM layers, 1 AE layer, 1 flow
    step), scaled to one full inference by the FLOP ratio."""
    from oracle import oracle as O
    from paper_2510_26742_b200.roofline import totals
    sample = cfg.replace(ve_layers=1, llm_layers=2, ae_layers=1, flow_steps=1)
    x = O.gen_inputs(sample, 1)
    t = time.perf_counter()
    O.port_forward(sample, x, threads=threads)
    dt = time.perf_counter() - t
    scale = totals(cfg)["flops"] / totals(sample)["flops"]
    return {"value": dt * scale * 1e3, "unit": "ms", "cores": threads, "kind": "port",
            "sample": (f"reduced-depth twin (1 VE / 2 LLM / 1 AE layer, 1 flow step, full widths, "
                       f"{cfg.views} views): {dt:.2f} s x FLOP ratio {scale:.1f}")}


def run_ours(args) -> None:
    import torch
    from paper_2510_26742_b200 import engine as E
    from paper_2510_26742_b200.config import default_config
    from paper_2510_26742_b200.inputs import gen_inputs
    from paper_2510_26742_b200.roofline import ae_weight_bytes, kv_cache_bytes, lower_bound_ms, measured_peaks, totals

    ws, rank, local = init_replicas(args.gpus)
    os.environ["PI0B_STAGING_THREADS"] = str(staging_threads(ws))
    # one GPU per rank; more ranks than GPUs (a functional run of the multi-rank path on a
    # 1-GPU box) share devices round-robin
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    cfg = default_config(views=args.views, prompt_tokens=args.prompt)
    eng = E.Engine(cfg, device=local)
    eng.gen_weights(1)
    # parity first: the seed-1 inputs of the committed golden, through the public call
    x1 = gen_inputs(cfg, 1)
    y = eng.run(x1["patches"], x1["state"], x1["noise"], x1.get("prompt"))  # captures the CUDA graph
    assert np.isfinite(y).all()
    par = golden_parity(cfg, y)
    if par is not None:
        par["max_abs"], par["rel"], par["rms_err"] = reduce_over_ranks([par["max_abs"], par["rel"], par["rms_err"]])
        par["cos"] = reduce_over_ranks([par["cos"]], op="min")[0]
    x = gen_inputs(cfg, 1 + rank)
    y = eng.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
    stream = torch.cuda.Stream()          # a real (non-legacy) stream: events and replays share it
    sh = stream.cuda_stream
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # 256 MB > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    torch.cuda.set_stream(stream)
    for _ in range(args.warmup):
        eng.replay(0, sh)
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for a, b in ev:
            flush.zero_()                      # L2 flush between timed iterations (outside events)
            a.record(stream)
            eng.replay(0, sh)
            b.record(stream)
        barrier()
    ms = np.array([a.elapsed_time(b) for a, b in ev])
    p50, p90, mean = float(np.median(ms)), float(np.percentile(ms, 90)), float(ms.mean())

    # end-to-end through the public API (host fp64 in, host fp64 out)
    e2e = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        eng.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
        if i >= args.warmup:
            e2e.append((time.perf_counter() - t0) * 1e3)
    e2e_p50 = float(np.median(e2e))

    p50, p90, mean, e2e_p50 = reduce_over_ranks([p50, p90, mean, e2e_p50])

    # Dominant kernel: the action-expert megakernel (one launch = all 10 flow steps; HBM-bound on
    # the weight stream).  Algorithmic bytes per launch = every AE weight byte once per flow step
    # + the LLM K/V cache it reads; timed alone with CUDA events on the engine stream.
    peaks = measured_peaks()
    ae_ms, _ = eng.time_node("ae.mega", reps=3)
    ae_bytes = ae_weight_bytes(cfg) * cfg.flow_steps + kv_cache_bytes(cfg) * cfg.flow_steps
    ae_gbs = ae_bytes / (ae_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_ae_mega.json")
    if os.path.exists(prof):
        traffic = json.load(open(prof)).get("dram_bytes_per_launch")
    # secondary: the LLM fused gated FFN GEMM (41% of all FLOPs), tensor-bound
    ffn_ms, _ = eng.time_node("llm.ffn", reps=3)
    L = cfg.prefix_tokens
    ffn_flops = 2.0 * L * cfg.llm_width * 2 * cfg.llm_mlp
    ffn_tf = ffn_flops / (ffn_ms * 1e-3) / 1e12
    lb = lower_bound_ms(cfg)
    tot = totals(cfg)
    n_kernels = eng.kernel_count(0)
    ve_shard = None
    if ws > 1 and not args.no_ve_shard:
        eng.close()          # frees this replica's HBM for the shard engine
        ve_shard = ve_shard_bench(cfg, ws, rank, local, min(args.steps, 100), args.warmup, p50)
    if rank != 0:
        return
    # bytes that cross PCIe per call: the patches go as bf16 (converted on the host, engine.cu
    # stage_patches_bf16), everything else as the caller's fp64
    in_bytes = sum(v.nbytes // 4 if k == "patches" else v.nbytes for k, v in x.items())
    line = {
        "metric": METRIC, "value": round(p50, 4), "unit": "ms", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(mean, 4), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (rtvla::gen_inputs seed 1+rank; gen_weights seed 1)",
        "config": {"workload": f"pi0 {cfg.views} views 224x224, prompt {cfg.prompt_tokens}, chunk 63, 10 flow steps",
                   "views": cfg.views, "prompt_tokens": cfg.prompt_tokens, "prefix_tokens": L,
                   "parallelism": f"replicas only ({ws} independent engines, no NCCL)" if ws > 1 else "single GPU",
                   "l2": "flushed (256 MB write) between timed replays; weights 5.2 GB >> 126 MB L2"},
        "p90_ms": round(p90, 4),
        "throughput_inf_per_s": round(ws * 1e3 / mean, 2),
        "e2e": {"value": round(e2e_p50, 4), "unit": "ms", "h2d_bytes_per_step": int(in_bytes),
                "d2h_bytes_per_step": int(y.nbytes)},
        "gpu_launches": n_kernels * args.steps,
        "gpu_launches_per_step": n_kernels,
        "roofline": {"bound": "hbm", "kernel": "action-expert megakernel (aemk_kernel, 1 launch = 10 flow steps)",
                     "achieved": round(ae_gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": round(ae_gbs / peaks["hbm_gbs"], 4), "traffic": traffic,
                     "bytes_per_launch": ae_bytes, "ms_per_launch": round(ae_ms, 4),
                     "share_of_step": round(ae_ms / mean, 3), "peak_source": peaks["source"] + " copy bandwidth"},
        "roofline_prefill_gemm": {"bound": "tensor", "kernel": "llm.ffn fused gated GEMM (tcgen05)",
                                  "achieved": round(ffn_tf, 1), "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                                  "frac": round(ffn_tf / peaks["bf16_tflops"], 4), "flops_per_launch": ffn_flops,
                                  "ms_per_launch": round(ffn_ms, 5), "peak_source": peaks["source"] + " burst"},
        "step_roofline": {"method": "reference lower bound sum max(2KM/BW, NKM/MAC) (costmodel.cpp:82-92)",
                          "lower_bound_ms": round(lb["total"], 4), "frac": round(lb["total"] / p50, 4),
                          "stages_ms": {k: round(v, 4) for k, v in lb.items() if k != "total"},
                          "flops": tot["flops"], "achieved_tflops": round(tot["flops"] / (p50 * 1e-3) / 1e12, 1)},
        "clocks": clk.summary(),
        "parity": par,
        "paper_4090_ms": {1: 20.0, 2: 27.3, 3: 36.8}.get(cfg.views),
    }
    if ve_shard is not None:
        line["ve_shard"] = ve_shard
    if ws == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline_port(cfg, os.cpu_count() or 1)
        except Exception as e:  # the baseline never blocks the GPU number
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)


def run_reference(args) -> None:
    """ONE full-scale rtvla::evaluate of the benched config (see the module docstring)."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2510_26742_b200.config import default_config
    cfg = default_config(views=args.views, prompt_tokens=args.prompt)
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/librtvla_ref.so not built"}))
        return
    t0 = time.perf_counter()
    ctx = O.RefContext(cfg)                 # build_pi0_graph + gen_weights + gen_inputs, seed 1
    setup_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    y = ctx.evaluate()                      # the reference's inference call (evaluate.cpp:365-370)
    ms = (time.perf_counter() - t0) * 1e3
    ctx.close()
    par = golden_parity(cfg, y)             # the reference against its own committed output
    cpu = ""
    try:
        cpu = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].split(":", 1)[1].strip()
    except Exception:
        pass
    line = {
        "metric": METRIC, "value": round(ms, 1), "unit": "ms", "n_gpus": ws, "steps": 1,
        "warmup": 0, "ms_per_step": round(ms, 1), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (gen_weights/gen_inputs seed 1)",
        "config": {"workload": f"pi0 {cfg.views} views 224x224, prompt {cfg.prompt_tokens}, chunk 63, 10 flow steps",
                   "views": cfg.views, "prompt_tokens": cfg.prompt_tokens, "prefix_tokens": cfg.prefix_tokens},
        "impl": "reference",
        "cpu_baseline": {"value": round(ms, 1), "unit": "ms", "cores": 1, "kind": "reference",
                         "sample": ("one full-scale rtvla::evaluate of this config (unmodified reference, -O3, "
                                    "single-threaded fp64: the reference has no internal parallelism); "
                                    f"setup (graph, gen_weights, gen_inputs) {setup_s:.1f} s untimed"),
                         "cpu": cpu, "nproc": os.cpu_count()},
        "e2e": {"value": round(ms, 1), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "parity": par,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--views", type=int, default=2)
    ap.add_argument("--prompt", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ve-shard", action="store_true", help="skip the view-sharded VE measurement at N > 1")
    ap.add_argument("--launch-check", action="store_true",
                    help="exercise the replica launcher + gloo reduction only (no GPU; tests/test_dist_cpu.py)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_replicas(sys.argv[1:], args.gpus))
    if args.launch_check:
        ws, rank, _ = init_replicas(args.gpus)
        hi = reduce_over_ranks([rank, 10.0 + rank])
        lo = reduce_over_ranks([rank], op="min")
        if rank == 0:
            print(json.dumps({"world_size": ws, "max": hi, "min": lo, "staging_threads": staging_threads(ws),
                              "nccl_initialized": _nccl_used()}), flush=True)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
