"""Benchmark: SpecPipe single-request time-between-tokens on B200.

Workload (BASELINE.json configs[1]): Llama-2-7B-shape random-init target
(LCG weights, fan-in scaled, bf16), 8 pipeline stages, single request,
dynamic tree w=64 / k=16, 512-token synthetic prompt, SyntheticDraft with
the paper-calibrated defaults (top1 0.62, decay 0.6, miss 0.01) bound to
the model's own greedy continuation.  With --gpus N the 8 stages are spread
over N GPUs (stage s on GPU s*N//8) and driven by one host process (the
reference's single-process design); other ranks only join the barriers.

  value   engine TBT: PipelineRunner.step on the recorded levels (draft cost
          excluded, level inputs staged), CUDA-event timed on the stream
  e2e     the public decode_step() path with the live draft, host buffers in
          and the verified token out every step (wall clock == event clock,
          the host blocks on the token each step)
  roofline  the tcgen05 weight-streaming GEMM (K2): algorithmic bytes
          (weights + node rows) / event-timed launch duration, averaged over
          every GEMM launch of a profiled replay of the timed steps
  cpu_baseline  the numpy restatement of the same step (oracle/llama.py,
          per-node float32 matvecs as the reference's layer_step) timed on a
          bounded sample and scaled to the measured node-layer count per step

--impl reference times that CPU restatement as the reference arm.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TBT ms/token (single request, 8-stage)"
UNIT = "ms/token"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=512)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="7b", choices=["7b", "13b", "70b", "tiny"])
    ap.add_argument("--stages", type=int, default=8)
    ap.add_argument("--prompt-len", type=int, default=512)
    ap.add_argument("--w", type=int, default=64)
    ap.add_argument("--k", type=int, default=16)
    ap.add_argument("--draft", default="paper", choices=["paper", "perfect"])
    ap.add_argument("--draft-model", default="auto", choices=["auto", "none", "68m", "7b"],
                    help="draft model whose forward runs each step (auto: 68m for 7b/13b targets, 7b for 70b)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--emulate-gpus", type=int, default=1,
                    help="diagnostics: the --gpus N placement (N shard objects, stage-per-GPU protocol on shard "
                         "streams) on GPU 0")
    ap.add_argument("--no-c1", action="store_true", help="skip the C1 leg vs the unmodified reference")
    ap.add_argument("--no-comparators", action="store_true", help="skip the vanilla-PP / cuBLAS comparators")
    ap.add_argument("--no-perfect", action="store_true", help="skip the perfect-draft TBT field")
    ap.add_argument("--profile-steps", type=int, default=24)
    ap.add_argument("--db-model", default="13b", choices=["7b", "13b", "70b", "tiny"])
    ap.add_argument("--db-batches", default="1,2,4,8,16,32,64", help="SpecPipe-DB batch sizes (empty: skip)")
    ap.add_argument("--db-new", type=int, default=24)
    return ap.parse_args()


def model_cfg(name):
    from paper_2504_04104_b200.model import LlamaConfig

    return {"7b": LlamaConfig.llama2_7b, "13b": LlamaConfig.llama2_13b, "70b": LlamaConfig.llama2_70b,
            "tiny": lambda: LlamaConfig(vocab=512, hidden=256, layers=8, heads=2, kv_heads=1, ffn=512)}[name]()


def draft_cfg(kind, seed=0):
    import paper_2504_04104_b200 as tp

    if kind == "perfect":
        return tp.SyntheticDraftConfig(top1_hit=1.0, rank_decay=0.5, miss_prob=0.0, seed=seed)
    return tp.SyntheticDraftConfig(seed=seed)


def draft_model_name(args):
    if args.draft_model != "auto":
        return None if args.draft_model == "none" else args.draft_model
    return {"70b": "7b", "tiny": None}.get(args.model, "68m")


def draft_model_cfg(name):
    from paper_2504_04104_b200.model import LlamaConfig

    return {"68m": LlamaConfig.llama_68m, "7b": lambda: LlamaConfig.llama2_7b(seed=1)}[name]()


def workload(args):
    dm = draft_model_name(args)
    return {"workload": f"Llama-2-{args.model}-shape target, {args.stages}-stage SpecPipe, single request, dynamic tree",
            "model": f"llama2-{args.model}-shape (random LCG init, fan-in scaled)", "stages": args.stages,
            "w": args.w, "k": args.k, "prompt_len": args.prompt_len, "draft": f"SyntheticDraft({args.draft})",
            "draft_model": (f"llama-{dm}-shape on stage 1's GPU: its tree forward over stage 1's level, LM head and "
                            "top-k run every step (timed); the host waits for the top-k before expanding"
                            if dm else None),
            "global_batch": 1, "parallelism": f"pp{args.stages} over {args.gpus} GPU(s)",
            "l2": "no flush: every step streams all stage weights (>>126 MB L2)",
            "untimed_before_warmup": f"a priming run of {2 * args.stages + 8} steps on a separate runner, then "
                                     f"{args.stages} pipeline-fill steps"}


class ClockSampler:
    """SM clock and throttle reasons sampled DURING a timed region, in-process
    through NVML (nvidia-ml-py; an nvidia-smi subprocess per sample perturbed
    the host loop it was measuring).  Falls back to nvidia-smi if NVML fails."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu=0, period=0.05):
        self.gpu, self.period, self.samples, self._stop = gpu, period, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(gpu)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:  # noqa: BLE001
            self._nvml = None
            self.max_mhz = None

    def _sample(self):
        if self._nvml is not None:
            nv = self._nvml
            sm = float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
            reasons = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))
            return sm, reasons
        out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        sm, mx = (float(x) for x in out.stdout.strip().split(","))
        self.max_mhz = mx
        return sm, 0

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        self._stop.clear()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ----------------------------------------------------------------------------- CPU arm


def cpu_step_estimate(cfg, node_layers_per_step, head_per_token, prompt_len, sample_nodes=8):
    """Time the numpy restatement on a bounded sample: `sample_nodes` tree-node
    forwards through one Llama layer (ctx = prompt_len) plus one LM-head row,
    then scale to the measured node-layer count of a step."""
    from oracle.llama import LlamaOracle, bf16
    from oracle.toy import OracleKv

    t_build = time.perf_counter()
    o = LlamaOracle(cfg.vocab, cfg.hidden, cfg.layers, cfg.heads, cfg.kv_heads, cfg.ffn, seed=cfg.seed,
                    layer_range=(0, 1), with_head=True)
    build_s = time.perf_counter() - t_build
    kvd = cfg.kv_heads * 128
    kv = OracleKv(cfg.layers, kvd)
    rng = np.random.default_rng(0)
    for p in range(prompt_len):  # synthetic prefix rows (values irrelevant to timing)
        kv.open_row(-1, p, True)
        kv.put(0, bf16(rng.standard_normal(kvd).astype(np.float32)), bf16(rng.standard_normal(kvd).astype(np.float32)))
    x = o.embed(1, prompt_len)
    rows = list(range(prompt_len))
    t0 = time.perf_counter()
    for i in range(sample_nodes):
        o.run_position(x, kv, rows, (0, 1), True, 10 + i, prompt_len)
    t_node_layer = (time.perf_counter() - t0) / sample_nodes
    t0 = time.perf_counter()
    o.greedy(x)
    t_head = time.perf_counter() - t0
    ms = (t_node_layer * node_layers_per_step + t_head * head_per_token) * 1e3
    return ms, {"t_node_layer_ms": t_node_layer * 1e3, "t_head_ms": t_head * 1e3, "build_s": build_s,
                "sample": f"{sample_nodes} node forwards through one {cfg.hidden}-wide layer (ctx {prompt_len}) + "
                          f"1 LM-head row, scaled to {node_layers_per_step:.0f} node-layers/step"}


class _ControlOnlyModel:
    """Stand-in model for a control-only run of the step machine: no compute, the
    verified token is read from a bound continuation.  The SyntheticDraft's hit
    pattern depends on whether its candidates contain the true next token, not on
    the token values, so a random continuation gives the workload's schedule
    (steps/token, resident nodes per stage) without the model's arithmetic."""

    def __init__(self, layers, truth, runner_ref):
        self.layers, self.hidden, self.truth, self._runner = layers, 1, truth, runner_ref

    def embed(self, token, pos):
        return np.zeros(1, np.float32)

    def run_position(self, x, kv, rows, layer_range=None, append=True, uid=-1, pos=0, prefix=False):
        if append:
            kv.open_row(uid, pos, prefix)
        return x

    def greedy(self, x):
        return int(self.truth[len(self._runner[0].verified)])


def run_reference(args):
    """The reference algorithm on the box's host cores (kind "port"): the step
    machine restated in oracle/pipeline.py (`pipeline.py:272-490`) over the float32
    Llama restatement with the reference's per-node forward_tree (one matvec chain
    per node and layer, `model.py:250-349`), at the full 7B shape, all 32 layers.

    Setup (untimed): weights from the LCG stream, a batched causal prompt prefill,
    the greedy continuation the SyntheticDraft binds to (`pipeline.py:599-602`),
    and the m-step pipeline fill.  Timed: min(K, 2) whole steady-state steps
    (10-30 s of CPU work; "steps" reports what ran).  ms/token = the measured time
    per node-layer x the node-layers per step x the steps per token, the last two
    measured in this process by a 512-step control-only run of the same step
    machine and draft (no constants)."""
    import copy

    import paper_2504_04104_b200 as tp
    from oracle.llama import LlamaOracle
    from oracle.pipeline import OracleRunner

    cfg = model_cfg(args.model)
    cores = os.cpu_count()
    t_setup = time.perf_counter()
    # schedule of this workload: control-only run of the same step machine + draft
    rng = np.random.default_rng(1)
    sched_steps = 512
    truth = [int(t) for t in rng.integers(0, cfg.vocab, args.prompt_len + sched_steps + 4 * args.stages)]
    ref_box = [None]
    stub = _ControlOnlyModel(cfg.layers, truth, ref_box)
    sdraft = tp.SyntheticDraft(draft_cfg(args.draft), cfg.vocab)
    sdraft.bind_reference(tuple(truth))
    sr = OracleRunner(stub, args.stages, args.w, args.k, sdraft)
    ref_box[0] = sr
    sr.prefill(truth[: args.prompt_len])
    for _ in range(args.stages):
        sr.decode_step()
    t0, nl_sched = len(sr.emitted), 0
    for _ in range(sched_steps):
        nl_sched += sum(len(st["res"]["uids"]) * (st["range"][1] - st["range"][0])
                        for st in sr.stages if st["res"] is not None)
        sr.decode_step()
    spt = sched_steps / max(1, len(sr.emitted) - t0)
    nl_per_step = nl_sched / sched_steps

    # the real port at the workload shape
    o = LlamaOracle(cfg.vocab, cfg.hidden, cfg.layers, cfg.heads, cfg.kv_heads, cfg.ffn, seed=cfg.seed)
    prompt = [int(t) for t in np.random.default_rng([0, 0]).integers(0, cfg.vocab, args.prompt_len)]
    timed = max(1, min(args.steps, 2))
    warm = min(args.warmup, 1)
    runner = OracleRunner(o, args.stages, args.w, args.k, None,
                          new_kv=lambda: o.new_dense_kv(args.prompt_len + 64 * (args.stages + 4)))
    runner.prefill(prompt, batched=True)
    # greedy continuation (sequential_decode) on copies of the prefilled caches
    n_truth = args.stages + warm + timed + args.stages + 2
    caches = [copy.deepcopy(st["kv"]) for st in runner.stages]
    cont = []
    pos = len(prompt)
    # the prefill already holds every prompt row: the last position's output is
    # recomputed (append=False, same-position rows excluded) as the pipeline's root
    # level does (`pipeline.py:264-266`, `model.py:335-338`)
    xl = o.embed(prompt[-1], pos - 1)
    for st, kv in zip(runner.stages, caches):
        rows = [i for i in range(len(kv)) if kv.positions[i] != pos - 1]
        xl = o.run_position(xl, kv, rows, st["range"], False, -1, pos - 1, True)
    for _ in range(n_truth):
        tok = o.greedy(xl)
        cont.append(tok)
        xl = o.embed(tok, pos)
        for st, kv in zip(runner.stages, caches):
            xl = o.run_position(xl, kv, list(range(len(kv))), st["range"], True, -1, pos, True)
        pos += 1
    del caches
    draft = tp.SyntheticDraft(draft_cfg(args.draft), cfg.vocab)
    draft.bind_reference(tuple(prompt) + tuple(cont))
    runner.draft = draft
    for _ in range(args.stages + warm):  # pipeline fill + warm-up
        runner.decode_step()
    setup_s = time.perf_counter() - t_setup
    step_ms, nls = [], []
    for _ in range(timed):
        nls.append(sum(len(st["res"]["uids"]) * (st["range"][1] - st["range"][0])
                       for st in runner.stages if st["res"] is not None))
        ts = time.perf_counter()
        runner.decode_step()
        step_ms.append((time.perf_counter() - ts) * 1e3)
    assert runner.emitted == cont[: len(runner.emitted)], "CPU port diverged from its own greedy decode"
    t_head = time.perf_counter()
    o.greedy(xl)
    head_ms = (time.perf_counter() - t_head) * 1e3
    per_nl = (sum(step_ms) - head_ms * timed) / max(1, sum(nls))
    ms_step = per_nl * nl_per_step + head_ms
    value = ms_step * spt
    sample = (f"{timed} whole steady-state steps of the port ({sum(nls)} node-layers, "
              f"{sum(step_ms) / 1e3:.1f} s), per-node float32 matvecs, {args.model} shape, all {cfg.layers} layers; "
              f"scaled by {nl_per_step:.0f} node-layers/step and {spt:.3f} steps/token from a "
              f"{sched_steps}-step control-only run in this process")
    line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": args.gpus, "steps": timed,
            "warmup": warm, "ms_per_step": round(float(np.mean(step_ms)), 2), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {**workload(args), "draft_model": (
                "not run by the CPU port: the draft's proposals come from the same SyntheticDraft; its forward "
                "(68M shape) is ~1 % of a 7B step's node-layer FLOPs") if draft_model_name(args) else None},
            "impl": "reference", "steps_per_token": round(spt, 4), "node_layers_per_step": round(nl_per_step, 1),
            "measured_steps_ms": [round(x, 1) for x in step_ms], "measured_node_layers": nls,
            "ms_per_node_layer": round(per_nl, 3), "head_ms": round(head_ms, 2), "setup_s": round(setup_s, 1),
            "cpu_baseline": {"value": round(value, 2), "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": round(value, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm


def build_shards(cfg, stages, ngpu, max_nodes, emulate=False):
    """One model object per GPU holding its stages' layers (stage s on GPU s*N/stages);
    ``emulate``: the same N shard objects all on GPU 0 (the stage-per-GPU protocol on
    one device, shard streams)."""
    from paper_2504_04104_b200.model import LlamaModel
    from paper_2504_04104_b200.pipeline import split_layers

    splits = split_layers(cfg.layers, stages)
    dev_of = [s * ngpu // stages for s in range(stages)]
    shards = {}
    for dev in sorted(set(dev_of)):
        mine = [splits[s] for s in range(stages) if dev_of[s] == dev]
        lo, hi = mine[0][0], mine[-1][1]
        shards[dev] = LlamaModel(cfg, device=0 if emulate else dev, max_nodes=max_nodes, layer_range=(lo, hi),
                                 with_embed=(lo == 0), with_head=(hi == cfg.layers))
    return [shards[dev_of[s]] for s in range(stages)], splits


def run_single_stage(args):
    """C3's 1-stage point: SpecPipe needs >= 2 stages (the reference's ConfigError), so
    m = 1 is the GPU greedy decode of the whole model (`sequential_decode`, reference
    `model.py:364-385`), steady-state ms/token as the difference of two
    decode lengths (prefill and first-use costs cancel), wall clock, synchronised."""
    import torch

    import paper_2504_04104_b200 as tp
    from paper_2504_04104_b200.model import LlamaModel

    torch.cuda.set_device(0)
    cfg = model_cfg(args.model)
    m = LlamaModel(cfg, max_nodes=64)
    prompt = [int(t) for t in np.random.default_rng([0, 0]).integers(0, cfg.vocab, args.prompt_len)]
    tp.sequential_decode(m, prompt, 8)  # untimed warm-up
    lens = (8, 8 + args.steps)
    ts = []
    with ClockSampler(0) as clocks:
        for n_tok in lens:
            torch.cuda.synchronize()
            t = time.perf_counter()
            tp.sequential_decode(m, prompt, n_tok)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
    ms = (ts[1] - ts[0]) * 1e3 / (lens[1] - lens[0])
    peak, peak_src = peaks()
    q_, kv_ = cfg.heads * cfg.head_dim, cfg.kv_heads * cfg.head_dim
    wbytes = 2.0 * (cfg.layers * (cfg.hidden * (q_ + 2 * kv_) + q_ * cfg.hidden + 3 * cfg.hidden * cfg.ffn)
                    + cfg.vocab * cfg.hidden)
    line = {"metric": "TBT ms/token (single request, 1 stage = GPU greedy decode)", "value": round(ms, 4),
            "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": 8, "ms_per_step": round(ms, 4),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": f"Llama-2-{args.model}-shape, 1 stage: sequential greedy decode (SpecPipe needs "
                                   ">= 2 stages)", "model": f"llama2-{args.model}-shape (random LCG init, fan-in scaled)",
                       "stages": 1, "prompt_len": args.prompt_len, "global_batch": 1},
            "tokens_per_s": round(1e3 / ms, 2),
            "step_roofline": {"bound": "hbm", "algorithmic_bytes_per_step": round(wbytes),
                              "ideal_ms_per_step": round(wbytes / (peak * 1e6), 4),
                              "frac": round(wbytes / (ms * 1e-3) / 1e9 / peak, 4), "peak": peak,
                              "note": "weights + LM head per token (KV rows omitted)"},
            "clocks": clocks.summary()}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world):
    import torch

    import paper_2504_04104_b200 as tp
    from paper_2504_04104_b200 import _lib
    from paper_2504_04104_b200.pipeline import PipelineConfig, PipelineRunner, sequential_decode_staged

    ngpu = args.gpus
    torch.cuda.set_device(0)
    cfg = model_cfg(args.model)
    t0 = time.perf_counter()
    emu = args.emulate_gpus > 1
    shards, splits = build_shards(cfg, args.stages, args.emulate_gpus if emu else ngpu, max_nodes=max(64, args.w),
                                  emulate=emu)
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t0
    prompt = [int(t) for t in np.random.default_rng([0, 0]).integers(0, cfg.vocab, args.prompt_len)]
    fill = args.stages  # untimed pipeline-fill steps before the W warm-up steps (the pipeline is m deep)
    pre = fill + args.warmup
    n_ref = pre + args.steps + args.profile_steps + 2 * args.stages + 16
    ref = sequential_decode_staged(shards if (ngpu > 1 or emu) else shards[0], splits, prompt, n_ref)
    pcfg = PipelineConfig(num_stages=args.stages, layer_splits=tuple(splits))
    beam = tp.BeamConfig(w=args.w, k=args.k)
    model_arg = shards if (ngpu > 1 or emu) else shards[0]
    dm_name = draft_model_name(args)
    dmodel = None
    if dm_name:
        from paper_2504_04104_b200.model import LlamaModel

        dmodel = LlamaModel(draft_model_cfg(dm_name), device=0, max_nodes=max(64, args.w))

    def fresh(draft, with_draft_model=True):
        r = PipelineRunner(model_arg, pcfg, beam, draft, collect_trace=False,
                           kv_capacity=args.prompt_len + n_ref + args.w * (args.stages + 2) + 64,
                           check_invariants=False, draft_model=dmodel if with_draft_model else None,
                           shard_streams=emu)
        r.prefill(prompt)
        return r

    streams = [torch.cuda.current_stream(d) for d in range(ngpu)]

    def joined(runner):
        """Device 0's current stream after every shard stream of ``runner`` (stage per GPU:
        the work runs on shard streams, so an end event must wait for them)."""
        for st in getattr(runner, "_shard_streams", None) or []:
            streams[0].wait_stream(st)
        return streams[0]

    def sync_all():
        for d in range(ngpu):
            torch.cuda.synchronize(d)

    # ---- priming (untimed initialisation): one throw-away run through the pipeline fill
    # and into steady state, so first-use growth (workspace slots, stage pools, staging
    # rings, larger levels) is not charged to the measured runs whatever W is
    pdraft0 = tp.SyntheticDraft(draft_cfg(args.draft), cfg.vocab)
    pdraft0.bind_reference(tuple(prompt) + tuple(ref))
    prime = fresh(pdraft0)
    for _ in range(min(2 * args.stages + 8, len(ref) // 2)):
        prime.decode_step()
    sync_all()
    prime.close()
    del prime

    # ---- e2e: public decode_step with the live draft ----------------------------------
    draft = tp.SyntheticDraft(draft_cfg(args.draft), cfg.vocab)
    draft.bind_reference(tuple(prompt) + tuple(ref))
    runner = fresh(draft)
    runner.children_log = []
    for _ in range(pre):  # pipeline fill, then the W warm-up steps
        runner.decode_step()
    sync_all()
    runner.host_s = {k: 0.0 for k in runner.host_s}
    tok0, steps0 = len(runner.emitted), runner.step_no
    l0 = _lib.launch_count()
    io0 = _lib.io_bytes()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    gc.collect()  # as timeit does: no cyclic-GC pause (or finaliser run) inside a timed loop
    gc.disable()
    with ClockSampler(0) as clocks:
        t_wall = time.perf_counter()
        ev[0].record(streams[0])
        for _ in range(args.steps):
            runner.decode_step()
        ev[1].record(joined(runner))
        sync_all()
        t_wall = time.perf_counter() - t_wall
    gc.enable()
    e2e_tokens = len(runner.emitted) - tok0
    e2e_ms = t_wall * 1e3 / max(1, e2e_tokens)
    e2e_host = {k: round(v * 1e3 / args.steps, 4) for k, v in runner.host_s.items()}
    e2e_host["loop_wall"] = round(t_wall * 1e3 / args.steps, 4)
    launches = _lib.launch_count() - l0
    io1 = _lib.io_bytes()
    for _ in range(args.profile_steps + 8):  # untimed: levels for the timeline (8) and profiled replays below
        runner.decode_step()
    resident = []
    children = runner.children_log
    assert runner.emitted == ref[: len(runner.emitted)], "SpecPipe output diverged from greedy decode"
    hit_rate = runner.hits / max(1, runner.hits + runner.misses)
    runner.close()
    del runner

    # ---- value: engine step on the recorded levels -----------------------------------
    replay = fresh(None)
    for ch in children[:pre]:
        replay.step(ch)
    sync_all()
    tok0 = len(replay.emitted)
    node_layers = 0
    step_bytes = 0.0  # SURVEY §8d algorithmic bytes of the timed steps
    q_, kv_ = cfg.heads * cfg.head_dim, cfg.kv_heads * cfg.head_dim
    layer_w = 2.0 * (cfg.hidden * (q_ + 2 * kv_) + q_ * cfg.hidden + 3 * cfg.hidden * cfg.ffn)
    head_w = 2.0 * cfg.vocab * cfg.hidden
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    replay.host_s = {k: 0.0 for k in replay.host_s}
    gc.collect()
    gc.disable()
    th = time.perf_counter()
    clocks.__enter__()
    e0.record(streams[0])
    for ch in children[pre : pre + args.steps]:
        node_layers += sum(len(s.resident) * (s.layer_range[1] - s.layer_range[0])
                           for s in replay.stages if s.resident is not None)
        resident.append([len(s.resident) if s.resident is not None else 0 for s in replay.stages])
        for s in replay.stages:
            if s.resident is None:
                continue
            nl, ns = s.layer_range[1] - s.layer_range[0], len(s.resident)
            ctx = len(s.kv)  # rows streamed once per layer (prefix + speculative)
            step_bytes += nl * (layer_w + ctx * 2 * kv_ * 2 + ns * 2 * kv_ * 2)
            if s.layer_range[0] == 0:
                step_bytes += ns * cfg.hidden * 2
            if s is replay.stages[-1]:
                step_bytes += head_w
        if dmodel is not None and replay.stages[0].resident is not None:  # the draft's weights, per step
            dc = dmodel.cfg
            dq, dkv = dc.heads * dc.head_dim, dc.kv_heads * dc.head_dim
            step_bytes += 2.0 * (dc.layers * (dc.hidden * (dq + 2 * dkv) + dq * dc.hidden + 3 * dc.hidden * dc.ffn)
                                 + dc.vocab * dc.hidden)
        replay.step(ch)
    e1.record(joined(replay))
    host_loop_s = time.perf_counter() - th
    sync_all()
    gc.enable()
    clocks.__exit__()
    host_diag = {k: round(v * 1e3 / args.steps, 4) for k, v in replay.host_s.items()}
    host_diag["loop_wall"] = round(host_loop_s * 1e3 / args.steps, 4)
    value_tokens = len(replay.emitted) - tok0
    value_ms = e0.elapsed_time(e1) / max(1, value_tokens)
    assert replay.emitted == ref[: len(replay.emitted)]

    no_draft_ms = None
    if dmodel is not None:  # the same replay without the draft model's forward (its cost on this GPU)
        nd = fresh(None, with_draft_model=False)
        for ch in children[:pre]:
            nd.step(ch)
        sync_all()
        ntok0 = len(nd.emitted)
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gc.collect()
        gc.disable()
        d0.record(streams[0])
        for ch in children[pre : pre + args.steps]:
            nd.step(ch)
        d1.record(joined(nd))
        sync_all()
        gc.enable()
        no_draft_ms = d0.elapsed_time(d1) / max(1, len(nd.emitted) - ntok0)
        nd.release()
        del nd

    # ---- GPU phase timeline of a few steps (diagnostic, separate from the timed run) -----
    replay.phase_events = []
    _lib.timeline_enable(True)
    _lib.timeline_read()
    for ch in children[pre + args.steps : pre + args.steps + 8]:
        replay.step(ch)
    sync_all()
    _lib.timeline_enable(False)
    kernel_tl = {k: round(v / 8, 4) for k, v in sorted(_lib.timeline_read().items(), key=lambda kv: -kv[1])}
    phases: dict[str, float] = {}
    evs = replay.phase_events
    for (ta, ea), (tb, eb) in zip(evs, evs[1:]):
        key = f"{ta}->{tb}"
        phases[key] = phases.get(key, 0.0) + ea.elapsed_time(eb)
    nsteps = max(1, sum(1 for t, _ in evs if t == "end"))
    phase_diag = {k: round(v / nsteps, 4) for k, v in phases.items()}
    replay.phase_events = None

    # ---- roofline: profiled replay of the next steps -------------------------------------
    _lib.profile_enable(True)
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record(streams[0])
    for ch in children[pre + args.steps + 8 :]:
        replay.step(ch)
    pe1.record(joined(replay))
    sync_all()
    _lib.profile_enable(False)
    by_members = _lib.profile_read_members()
    gemm_ms = sum(r[0] for r in by_members)
    gemm_bytes = sum(r[1] for r in by_members)
    gemm_n = sum(r[2] for r in by_members)
    prof_total_ms = pe0.elapsed_time(pe1)
    peak, peak_src = peaks()
    achieved = gemm_bytes / (gemm_ms * 1e-3) / 1e9 if gemm_ms > 0 else 0.0
    try:  # measured DRAM traffic of the same kernel (committed ncu capture, see profiles/)
        with open(os.path.join(ROOT, "profiles", "r02f_gemm_traffic.json")) as fh:
            cap = json.load(fh)
    except Exception:  # noqa: BLE001
        cap = None

    steps_per_token = args.steps / max(1, e2e_tokens)
    per_step_h2d = (io1[0] - io0[0]) / args.steps
    per_step_d2h = (io1[1] - io0[1]) / args.steps
    line = {
        "metric": METRIC, "value": round(value_ms, 4), "unit": UNIT, "n_gpus": ngpu, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(value_ms / steps_per_token, 4), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": workload(args),
        "tokens_per_s": round(1e3 / value_ms, 2),
        "e2e": {"value": round(e2e_ms, 4), "unit": UNIT, "h2d_bytes_per_step": int(per_step_h2d),
                "d2h_bytes_per_step": int(per_step_d2h), "tokens_per_s": round(1e3 / e2e_ms, 2)},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "sk_gemm_kernel (tcgen05 weight-streaming GEMM)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4),
                     "traffic": cap["traffic_bytes_per_launch"] if cap else None,
                     "traffic_capture": ({**{k: cap[k] for k in ("launches", "algorithmic_bytes_per_launch",
                                                                 "traffic_over_algorithmic", "source")},
                                          "note": "a separate ncu capture of the same workload (profiles/); compare "
                                                  "traffic with its own algorithmic_bytes_per_launch, not with this "
                                                  "run's bytes_per_launch"}
                                         if cap else None),
                     "peak_source": peak_src,
                     "gemm_share_of_step": round(gemm_ms / prof_total_ms, 4) if prof_total_ms else None,
                     "gemm_launches": gemm_n, "bytes_per_launch": round(gemm_bytes / max(1, gemm_n)),
                     "by_members": {str(i + 1): {"launches": r[2], "frac": round(r[1] / (r[0] * 1e-3) / 1e9 / peak, 4),
                                                 "ms_per_step": round(r[0] / max(1, len(children[pre + args.steps + 8:])), 4)}
                                    for i, r in enumerate(by_members) if r[2]},
                     "by_members_note": "launches by member count: the grouped stage forwards (3+ members), the "
                                        "verify stage (+ the fused draft model: 2), the LM heads (1)"},
        "step_roofline": {"bound": "hbm", "algorithmic_bytes_per_step": round(step_bytes / max(1, len(resident))),
                          "ideal_ms_per_step": round(step_bytes / max(1, len(resident)) / (peak * 1e6), 4),
                          "achieved": round(step_bytes / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1),
                          "frac": round(step_bytes / (e0.elapsed_time(e1) * 1e-3) / 1e9 / peak, 4),
                          "unit": "GB/s", "note": "whole engine step (all kernels + host gaps) vs weights of the "
                                                  "occupied stages + KV rows + LM head, per SURVEY 8d"},
        "draft_model_cost": ({"tbt_ms_per_token_without": round(no_draft_ms, 4),
                              "share": round(1 - no_draft_ms / value_ms, 4),
                              "note": "the same replayed steps without the draft model's forward (engine value)"}
                             if no_draft_ms else None),
        "host_ms_per_step": host_diag,
        "e2e_host_ms_per_step": e2e_host,
        "gpu_phase_ms_per_step": phase_diag,
        "gpu_kernel_ms_per_step": kernel_tl,
        "clocks": clocks.summary(),
        "steps_per_token": round(steps_per_token, 4), "hit_rate": round(hit_rate, 4),
        "mean_resident_nodes": [round(float(x), 2) for x in np.mean(np.asarray(resident), axis=0)] if resident else None,
        "node_layers_per_step": round(node_layers / max(1, len(resident)), 1),
        "init_s": round(init_s, 1),
    }
    if rank == 0 and ngpu == 1 and not args.no_cpu_baseline:
        ms, info = cpu_step_estimate(cfg, node_layers / max(1, len(resident)), 1.0, args.prompt_len)
        line["cpu_baseline"] = {"value": round(ms * steps_per_token, 2), "unit": UNIT, "cores": os.cpu_count(),
                                "kind": "port", "sample": info["sample"]}
    if args.draft == "paper" and not args.no_perfect:
        # the same engine with a perfect draft (every verification hits): steps/token -> 1,
        # isolating system overhead against the one-token-per-pipeline-step bound
        pdraft = tp.SyntheticDraft(draft_cfg("perfect"), cfg.vocab)
        pdraft.bind_reference(tuple(prompt) + tuple(ref))
        pr = fresh(pdraft)
        for _ in range(args.stages + args.warmup):  # pipeline fill + W warm-up steps
            pr.decode_step()
        sync_all()
        pt0 = len(pr.emitted)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gc.collect()
        gc.disable()
        f0.record(streams[0])
        nsteps = min(args.steps, max(8, len(ref) - len(pr.emitted) - args.stages - 2))
        for _ in range(nsteps):
            pr.decode_step()
        f1.record(joined(pr))
        sync_all()
        gc.enable()
        ptok = len(pr.emitted) - pt0
        assert pr.emitted == ref[: len(pr.emitted)]
        line["perfect_draft"] = {"tbt_ms_per_token": round(f0.elapsed_time(f1) / max(1, ptok), 4),
                                 "steps": nsteps, "tokens": ptok,
                                 "ms_per_step": round(f0.elapsed_time(f1) / nsteps, 4),
                                 "ideal_ms_per_step_all_stages_occupied": round(
                                     (args.stages * (cfg.layers // args.stages) * layer_w + head_w) / (peak * 1e6), 4)}
        pr.close()
    if rank == 0 and line.get("mean_resident_nodes"):
        line["per_stage"] = stage_profile(args, cfg, model_arg, splits, line["mean_resident_nodes"],
                                          args.prompt_len + int(round(e2e_tokens / 2)), steps_per_token, peak)
    if not args.no_comparators:
        line["comparators"] = comparators(args, cfg, model_arg, splits, prompt, sync_all)
    if rank == 0 and ngpu == 1 and args.db_batches:
        line["specpipe_db"] = run_db(args)
    if rank == 0 and ngpu == 1 and not args.no_c1:
        line["c1_vs_reference"] = c1_leg()
    print(json.dumps(line), flush=True)


def stage_profile(args, cfg, model_arg, splits, mean_nodes, ctx, steps_per_token, peak, iters=20):
    """Each stage's lone forward at its steady-state node count (rounded mean
    resident nodes of the timed steps) over a `ctx`-row cache, timed with CUDA
    events — what one stage per GPU would run every step (the last stage with K4
    verify).  SURVEY 8d per-stage bytes (weights of its layers + prefix K/V +
    new K/V rows + [first] embeddings + [last] LM head) over that time gives the
    per-stage roofline fraction; max over stages x steps/token is the projected
    stage-per-GPU TBT (a projection from one-GPU measurements, not a multi-GPU
    run)."""
    import torch

    import paper_2504_04104_b200 as tp
    from paper_2504_04104_b200.model import forward_members
    from paper_2504_04104_b200.pipeline import PipelineConfig, PipelineRunner

    depth = 12
    rng = np.random.default_rng(5)
    prompt = [int(t) for t in rng.integers(0, cfg.vocab, ctx + depth)]
    r = PipelineRunner(model_arg, PipelineConfig(num_stages=args.stages, layer_splits=tuple(splits)),
                       tp.BeamConfig(w=args.w, k=args.k), None, collect_trace=False, kv_capacity=ctx + depth + 128,
                       check_invariants=False)
    r.prefill(prompt)
    q_, kv_ = cfg.heads * cfg.head_dim, cfg.kv_heads * cfg.head_dim
    layer_w = 2.0 * (cfg.hidden * (q_ + 2 * kv_) + q_ * cfg.hidden + 3 * cfg.hidden * cfg.ffn)
    out = []
    for si, stage in enumerate(r.stages):
        n = max(1, int(round(mean_nodes[si])))
        dev = stage.model.device
        d = rng.integers(0, depth, n)
        pre = np.full(n, ctx, dtype=np.int32)
        bits = ((np.uint64(1) << d.astype(np.uint64)) - np.uint64(1)).reshape(n, 1).astype(np.uint64)
        with torch.cuda.device(dev):
            x = torch.randn(n, cfg.hidden, device=f"cuda:{dev}") * 0.5  # fp32 residual-stream rows
            item = (stage.kv, stage.model, x, None, (ctx + d).tolist(), stage.layer_range, False, list(range(n)),
                    False, (pre, ctx, 1, bits))
            last = si == len(r.stages) - 1

            def once():
                # K4 enqueued, its 16-byte result read by the host once per forward: on its own GPU
                # the verify stage's next forward does not wait for that read (the pipeline reads
                # it while the GPU goes on), so the wait is not inside the timed sequence
                o = forward_members([[item]])[0]
                if last:
                    stage.model.verify_async(o[0][0:1] if isinstance(o, list) else o[0:1])

            for _ in range(3):
                once()
                if last:
                    stage.model.verify_wait()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(iters):
                once()
            e1.record()
            torch.cuda.synchronize(dev)
            if last:
                stage.model.verify_wait()
        ms = e0.elapsed_time(e1) / iters
        nl = stage.layer_range[1] - stage.layer_range[0]
        b = nl * (layer_w + (ctx + depth) * 2 * kv_ * 2 + n * 2 * kv_ * 2)
        if stage.layer_range[0] == 0:
            b += n * cfg.hidden * 2
        if last:
            b += 2.0 * cfg.vocab * cfg.hidden
        out.append({"stage": si + 1, "nodes": n, "layers": nl, "ms": round(ms, 4), "bytes": int(b),
                    "frac": round(b / (ms * 1e-3) / 1e9 / peak, 4)})
    r.close()
    worst = max(x["ms"] for x in out)
    return {"stages": out, "ctx": ctx,
            "stage_per_gpu_projection": {"ms_per_step": worst, "tbt_ms_per_token": round(worst * steps_per_token, 4),
                                         "note": "projection: slowest measured lone stage x measured steps/token "
                                                 "(one stage per GPU, transfers overlapped); not a multi-GPU run"},
            "note": "each stage's lone forward (ungrouped launch sequence, last stage + K4 verify) at its rounded "
                    "mean resident node count, CUDA events, warm"}


def c1_leg(tokens=32):
    """BASELINE config 1 (the reference's own CPU demo shape): ToyModel V=64, d=256,
    L=4 (float64), 2 stages, paper beam w=64/k=16 and CLI beam w=4/k=4, 128-token
    prompt, SyntheticDraft paper defaults.  The UNMODIFIED reference (baseline/_ref,
    its own PipelineRunner, numpy on this box's host cores) and this package's B200
    path decode the same request; the decode loop (decode_step until `tokens` are
    emitted) is timed on both, after the untimed draft binding and prefill."""
    import importlib

    import torch

    import paper_2504_04104_b200 as tp

    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "treepipe")):
        return {"unavailable": "reference not installed under baseline/_ref"}
    sys.path.insert(0, ref_dir)
    try:
        ref = importlib.import_module("treepipe")
        refp = importlib.import_module("treepipe.pipeline")
    finally:
        sys.path.remove(ref_dir)
    prompt = [int(t) for t in np.random.default_rng([0, 0]).integers(0, 64, 128)]
    out = {"config": "C1: ToyModel V64 d256 L4 f64, 2 stages, prompt 128", "tokens": tokens,
           "reference_cores": os.cpu_count(), "results": []}
    rmodel = ref.init_model(ref.ToyModelConfig(vocab=64, hidden=256, layers=4, seed=0))
    gmodel = tp.init_model(tp.ToyModelConfig(vocab=64, hidden=256, layers=4, seed=0))
    truth = ref.sequential_decode(rmodel, prompt, tokens + 8)
    for w, k in ((64, 16), (4, 4)):
        row = {"w": w, "k": k}
        for impl, mod, model, Runner in (("reference", ref, rmodel, refp.PipelineRunner),
                                         ("b200", tp, gmodel, tp.PipelineRunner)):
            draft = mod.SyntheticDraft(mod.SyntheticDraftConfig(seed=0), 64)
            draft.bind_reference(tuple(prompt) + tuple(truth))
            r = Runner(model, mod.PipelineConfig(num_stages=2), mod.BeamConfig(w=w, k=k), draft,
                       collect_trace=False)
            r.prefill(prompt)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            while len(r.emitted) < tokens:
                r.decode_step()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            row[impl] = {"ms_per_token": round(dt * 1e3 / len(r.emitted), 4), "steps": r.step_no,
                         "steps_per_token": round(r.metrics().steps_per_token, 4)}
            row[impl + "_tokens"] = list(r.emitted)
        row["tokens_identical"] = row.pop("reference_tokens") == row.pop("b200_tokens")
        row["speedup"] = round(row["reference"]["ms_per_token"] / row["b200"]["ms_per_token"], 2)
        out["results"].append(row)
    return out


def comparators(args, cfg, model_arg, splits, prompt, sync_all):
    """SURVEY 8(d) GPU comparators on the same box and kernels:
    * vanilla PP (`run_vanilla` semantics, reference `pipeline.py:616-662`): one token
      in flight through every stage = steady-state GPU greedy decode of the staged
      model, timed as the difference of two decode lengths (the prefill cancels);
    * K2 vs cuBLAS (torch bf16 matmul) at the same tiny M: each layer GEMM of the
      model for the stage-1 mean node count and for the lone verify node."""
    import ctypes as C

    import torch

    from paper_2504_04104_b200 import _lib
    from paper_2504_04104_b200.pipeline import sequential_decode_staged

    out = {}
    lens = (8, 40)
    ts = []
    for n_tok in lens:
        sync_all()
        t = time.perf_counter()
        sequential_decode_staged(model_arg, splits, prompt, n_tok)
        sync_all()
        ts.append(time.perf_counter() - t)
    out["vanilla_pp"] = {"ms_per_token": round((ts[1] - ts[0]) * 1e3 / (lens[1] - lens[0]), 4),
                         "note": "same kernels at n=1, one token in flight through all stages (wall clock, "
                                 "synchronised, difference of a %d- and a %d-token decode)" % lens}
    lib = _lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    d, f = cfg.hidden, cfg.ffn
    q = cfg.heads * 128
    kvd = cfg.kv_heads * 128
    shapes = [("qkv", q + 2 * kvd, d), ("o", d, q), ("gate_up", 2 * f, d), ("down", d, f)]
    rows = []
    for n in (45, 1):
        for name, n_out, k in shapes:
            w = (torch.randn(n_out, k, device="cuda") * 0.02).to(torch.bfloat16)
            x = torch.randn(n, k, device="cuda").to(torch.bfloat16)
            y = torch.empty(n, n_out, device="cuda")
            ms = C.c_float()
            arr = lambda t: (C.c_void_p * 1)(t.data_ptr())  # noqa: E731
            _lib.check(lib.tp_debug_gemm_group_timed(0, 1, arr(w), arr(x), (C.c_int32 * 1)(n), n_out, k, arr(y),
                                                     20, C.byref(ms), st))
            for _ in range(3):
                torch.matmul(x, w.t())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                torch.matmul(x, w.t())
            e1.record()
            torch.cuda.synchronize()
            by = n_out * k * 2 + n * k * 2
            rows.append({"gemm": name, "n": n, "k2_us": round(ms.value * 1e3, 1),
                         "cublas_us": round(e0.elapsed_time(e1) * 1e3 / 20, 1),
                         "k2_gbs": round(by / ms.value / 1e6), "cublas_gbs": round(by / (e0.elapsed_time(e1) / 20) / 1e6)})
            del w, x, y
    out["k2_vs_cublas"] = rows
    return out


def run_db(args):
    """SpecPipe-DB (BASELINE config 5) on the same GPU: 13B-shape target, 8 stages,
    total tree width 64, FIFO requests all arriving at tick 0; steady-state
    tokens/s over the ticks where the whole batch is active (wall clock,
    synchronised; host scheduling included)."""
    import gc

    import torch

    from paper_2504_04104_b200.model import LlamaModel
    from scripts.bench_db import measure_db

    gc.collect()
    torch.cuda.empty_cache()
    # max_nodes 256: admission prefill of several requests in combined 256-row forwards
    model = LlamaModel(model_cfg(args.db_model), max_nodes=256)
    out = {"metric": "SpecPipe-DB tokens/s", "model": f"llama2-{args.db_model}-shape", "stages": 8,
           "total_width": 64, "k": 16, "prompt_len": args.prompt_len, "new_tokens": args.db_new, "results": []}
    batches = [int(x) for x in args.db_batches.split(",") if x]
    # untimed warm-up at the largest batch: workspace / stage-pool growth and first-use
    # costs otherwise land in the first measured session's steady-state ticks
    measure_db(model, min(16, max(batches)), args.prompt_len, 8)
    for b in batches:
        out["results"].append(measure_db(model, b, args.prompt_len, args.db_new))
    del model
    return out


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
        pg = dist
    try:
        if rank == 0:
            if args.impl == "reference":
                run_reference(args)
            elif args.stages == 1:
                run_single_stage(args)
            else:
                run_ours(args, rank, world)
    finally:
        if pg is not None:
            pg.barrier()
            pg.destroy_process_group()


if __name__ == "__main__":
    main()
