"""Record golden episode fixtures from the REFERENCE implementation.

Run in the build container only (it imports the read-only reference from
``/root/reference/pkg/src``); the fixtures it writes are committed and are
what the oracle and the CUDA path are pinned against on machines where the
reference is absent:

    python tests/golden/make_golden.py

For each case it builds a reference ``TuningSession`` (tuner.py:241-312),
warms its GBT cost model exactly like the survey's probe procedure (uniform
states from an independent generator, ``SimulatedBackend`` defaults,
``observe`` + ``fit_round``, costmodel.py:163-215), snapshots the session
state, then runs ``_run_episode`` (tuner.py:350-440) with light
instrumentation (wrapping the names ``select_actions``/``advantage``/
``ppo_update`` inside ``schedtune.tuner``) and records every per-step
quantity.  Large arrays are stored as SHA-256 digests of their bytes; the
oracle reproduces them bit for bit, so digests are enough.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

BMM_SOFTMAX_YAML = """
name: bert-attention
subgraphs:
  - id: bgemm_softmax
    weight: 12
    nodes:
      - name: bmm
        kind: batch_matmul
        shape: {b: 12, m: 128, k: 64, n: 128}
        consumers: [sm]
      - name: sm
        kind: softmax
        shape: {heads: 12, q: 128, k: 128}
"""


def digest(a) -> str:
    a = np.ascontiguousarray(np.asarray(a))
    h = hashlib.sha256()
    h.update(str(a.dtype.str).encode() + str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def digest_list(arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(digest(a).encode())
    return h.hexdigest()


CASES = [
    # name, workload (file or inline), subgraph index, target, cfg, episodes
    # (sketch index per episode), searcher, warm examples
    dict(name="gemm64_l2", workload="gemm_64.yaml", sg=0,
         target=dict(tiling_levels=2),
         cfg=dict(min_tracks=8, initial_tracks=16, cull_window=3,
                  episode_len=6, hidden=(16,), minibatch=32,
                  buffer_capacity=64, seed=5),
         sketches=[0, 2], searcher="rl", warm=64),
    dict(name="gemm64_fixed", workload="gemm_64.yaml", sg=0,
         target=dict(tiling_levels=2),
         cfg=dict(min_tracks=8, initial_tracks=16, cull_window=3,
                  episode_len=4, hidden=(16,), minibatch=16,
                  buffer_capacity=256, seed=9),
         sketches=[1], searcher="rl-fixed-length", warm=48),
    dict(name="gemm64_evo", workload="gemm_64.yaml", sg=0,
         target=dict(tiling_levels=2),
         cfg=dict(min_tracks=4, initial_tracks=8, cull_window=3,
                  episode_len=4, hidden=(16,), seed=2),
         sketches=[2], searcher="evolutionary", warm=32),
    dict(name="conv2d_l4", workload="conv2d.yaml", sg=2,
         target=dict(), cfg=dict(min_tracks=16, initial_tracks=32,
                                 cull_window=3, episode_len=6,
                                 hidden=(32, 32), minibatch=64,
                                 buffer_capacity=128, seed=1),
         sketches=[0, 1], searcher="rl", warm=96),
    dict(name="bmm_softmax_k3", workload=BMM_SOFTMAX_YAML, sg=0,
         target=dict(), cfg=dict(min_tracks=8, initial_tracks=16,
                                 cull_window=2, episode_len=4,
                                 hidden=(128, 128), minibatch=16,
                                 buffer_capacity=48, seed=3),
         sketches=[3, 0], searcher="rl", warm=64),
    dict(name="gpu_gemm1024", workload="gemm_l.yaml", sg=0,
         target="gpu", cfg=dict(min_tracks=8, initial_tracks=16,
                                cull_window=3, episode_len=4,
                                hidden=(32,), minibatch=16, seed=4),
         sketches=[0], searcher="rl-greedy-subgraph", warm=64),
]


def main():
    sys.path.insert(0, REF)
    import schedtune.tuner as T
    from schedtune.measure import MeasureRequest, SimulatedBackend
    from schedtune.schedspace import sample_initial_schedules
    from schedtune.tuner import SearcherKind, TunerConfig, TuningSession
    from schedtune.workload import TargetConfig, gpu_target, load_network

    wl_dir = "/root/reference/pkg/workloads"
    index = {}
    for case in CASES:
        wl = case["workload"]
        if wl.endswith(".yaml"):
            yaml_text = open(os.path.join(wl_dir, wl)).read()
        else:
            yaml_text = wl
        tmp = os.path.join("/tmp", f"golden_{case['name']}.yaml")
        with open(tmp, "w") as fh:
            fh.write(yaml_text)
        net = load_network(tmp)
        target = gpu_target() if case["target"] == "gpu" else \
            TargetConfig(**case["target"])
        cfg = TunerConfig(**case["cfg"])
        session = TuningSession(net, target, cfg, SimulatedBackend(),
                                SearcherKind(case["searcher"]))
        sg = net.subgraphs[case["sg"]]
        agent = session.agents[sg.id]
        rec = {"name": case["name"], "yaml": yaml_text, "sg": case["sg"],
               "target": (dict(name="gpu") if case["target"] == "gpu"
                          else case["target"]),
               "cfg": {k: (list(v) if isinstance(v, tuple) else v)
                       for k, v in case["cfg"].items()},
               "searcher": case["searcher"],
               "slots": session.slots[sg.id],
               "init_policy_digest": digest_list(agent.policy.params()),
               "init_value_digest": digest_list(agent.value.params()),
               "episodes": []}

        # -- warm the surrogate (independent generator, probe procedure) --
        wrng = np.random.default_rng(1000 + cfg.seed)
        backend = SimulatedBackend()
        for k_i, sk in enumerate(session.sketches[sg.id]):
            ctx = session.contexts[sk.id]
            states = sample_initial_schedules(sk, case["warm"], wrng)
            res = backend.measure_batch([MeasureRequest(s, ctx)
                                         for s in states])
            for s, r in zip(states, res):
                session.model.observe(ctx.featurize(s), r.throughput, sg.id)
        ex = session.model.training_examples()
        session.model.fit_round()
        trees = session.model.trees
        arrays = {}
        # the refit's training set (GBT refit parity, costmodel.py:190-212)
        arrays["fit_X"] = np.stack([e.features for e in ex])
        arrays["fit_y"] = np.asarray([e.target for e in ex], np.float64)
        arrays["model_base"] = np.asarray([session.model.base])
        for i, tr in enumerate(trees):
            arrays[f"tree{i:03d}_feature"] = tr.feature.astype(np.int16)
            arrays[f"tree{i:03d}_threshold"] = tr.threshold
            arrays[f"tree{i:03d}_left"] = tr.left.astype(np.int16)
            arrays[f"tree{i:03d}_right"] = tr.right.astype(np.int16)
            arrays[f"tree{i:03d}_value"] = tr.value
        rec["n_trees"] = len(trees)
        rec["model_lr"] = session.model.cfg.learning_rate

        orig = {n: getattr(T, n) for n in ("select_actions", "advantage",
                                           "ppo_update")}
        for e_i, sk_idx in enumerate(case["sketches"]):
            sketch = session.sketches[sg.id][sk_idx]
            ep = {"sketch": sk_idx,
                  "rng_state": session.rng.bit_generator.state,
                  "order_counter": session.order_counter,
                  "buffer_len": len(session.buffers[sg.id]),
                  "pi_t": agent.opt_pi.t, "v_t": agent.opt_v.t,
                  "policy_digest": digest_list(agent.policy.params()),
                  "value_digest": digest_list(agent.value.params()),
                  "steps": []}
            steps = ep["steps"]

            def sel_wrap(policy, X, masks, rng):
                acts, logp = orig["select_actions"](policy, X, masks, rng)
                steps.append({"X": digest(X), "masks": digest_list(masks),
                              "m": len(X)})
                arrays[f"e{e_i}_s{len(steps)}_actions"] = acts.astype(np.int16)
                arrays[f"e{e_i}_s{len(steps)}_logp"] = logp
                return acts, logp

            def adv_wrap(r, vn, vc, disc):
                out = orig["advantage"](r, vn, vc, disc)
                s = len(steps)
                arrays[f"e{e_i}_s{s}_rewards"] = r
                arrays[f"e{e_i}_s{s}_v_next"] = vn
                arrays[f"e{e_i}_s{s}_v_cur"] = vc
                arrays[f"e{e_i}_s{s}_adv"] = out
                return out

            def ppo_wrap(policy, value, opt_pi, opt_v, batch, rlcfg):
                out = orig["ppo_update"](policy, value, opt_pi, opt_v,
                                         batch, rlcfg)
                steps[-1]["ppo"] = {k: float(v) for k, v in out.items()}
                steps[-1]["ppo_policy_digest"] = digest_list(policy.params())
                steps[-1]["ppo_value_digest"] = digest_list(value.params())
                return out

            orig_uniform = session._uniform_actions

            def uni_wrap(masks):
                acts = orig_uniform(masks)
                steps.append({"masks": digest_list(masks),
                              "m": len(masks[0])})
                arrays[f"e{e_i}_s{len(steps)}_actions"] = acts.astype(np.int16)
                return acts

            T.select_actions, T.advantage, T.ppo_update = \
                sel_wrap, adv_wrap, ppo_wrap
            session._uniform_actions = uni_wrap
            try:
                entries = session._run_episode(sg, sketch, e_i + 1)
            finally:
                for n, f in orig.items():
                    setattr(T, n, f)
                del session._uniform_actions
            ctxt = session.contexts[sketch.id]
            L = sketch.space.levels
            tiles = np.asarray([[f for d in e.state.tiles for f in d]
                                for e in entries], dtype=np.uint16)
            knobs = np.asarray([[e.state.compute_at_index,
                                 e.state.parallel_fuse_count,
                                 e.state.unroll_index] for e in entries],
                               dtype=np.uint8)
            arrays[f"e{e_i}_entry_tiles"] = tiles.reshape(len(entries), -1) \
                if len(entries) else np.zeros((0, 0), np.uint16)
            arrays[f"e{e_i}_entry_knobs"] = knobs
            arrays[f"e{e_i}_entry_score"] = session.model.predict(
                np.stack([e.features for e in entries]))
            ep["entries_features_digest"] = digest(
                np.stack([e.features for e in entries]))
            ep["entries_canonical_digest"] = hashlib.sha256(
                "\n".join(e.canonical for e in entries).encode()).hexdigest()
            ep["entries_order"] = [entries[0].order, entries[-1].order,
                                   len(entries)]
            # rank_scores (costmodel.py:266-286) on these entries: several k,
            # with and without an exclude set of already-measured states
            from schedtune.costmodel import rank_scores
            distinct = list(dict.fromkeys(e.canonical for e in entries))
            excl = set(distinct[::5]) | set(
                e.canonical for e in rank_scores(session.model, entries, 3))
            ep["rank"] = []
            for k in (1, 8, 64, len(entries) + 5):
                for ex in (None, excl):
                    chosen = rank_scores(session.model, entries, k,
                                         exclude=ex)
                    ep["rank"].append({
                        "k": k,
                        "exclude": sorted(ex) if ex else [],
                        "chosen": [e.order for e in chosen]})
            ep["end_rng_state"] = session.rng.bit_generator.state
            ep["end_policy_digest"] = digest_list(agent.policy.params())
            ep["end_value_digest"] = digest_list(agent.value.params())
            ep["end_adam_digest"] = digest_list(agent.opt_pi.m + agent.opt_pi.v
                                                + agent.opt_v.m + agent.opt_v.v)
            ep["end_pi_t"] = agent.opt_pi.t
            ep["end_buffer_len"] = len(session.buffers[sg.id])
            ep["end_order_counter"] = session.order_counter
            ep["feature_len"] = ctxt.feature_len
            ep["levels"] = L
            rec["episodes"].append(ep)
        path = os.path.join(HERE, f"{case['name']}.npz")
        np.savez_compressed(path, **arrays)
        with open(os.path.join(HERE, f"{case['name']}.json"), "w") as fh:
            json.dump(rec, fh, indent=1, sort_keys=True,
                      default=lambda o: int(o) if isinstance(o, np.integer)
                      else str(o))
        index[case["name"]] = os.path.getsize(path)
        print(case["name"], "episodes", len(rec["episodes"]),
              "npz bytes", os.path.getsize(path))
    index["gbt_fit_large"] = make_gbt_fixture()
    index["sim"] = make_sim_fixture()
    return index


def make_sim_fixture():
    """The reference's analytic model: simulate_time of random states of
    several sketches (default and custom SimHwParams) and brute_force_best
    on the 4,116-state GEMM-64 space."""
    sys.path.insert(0, REF)
    from dataclasses import asdict
    from schedtune.measure import SimHwParams, brute_force_best, simulate_time
    from schedtune.schedspace import SketchContext, sample_initial_schedules
    from schedtune.workload import (TargetConfig, generate_sketches,
                                    gpu_target, load_network)
    wl_dir = "/root/reference/pkg/workloads"
    custom = SimHwParams(cores=8, cap_l1=2048.0, cap_l2=65536.0,
                         miss_penalty_l1=0.45, miss_penalty_l2=0.9,
                         parallel_overhead=0.05, peak_flops=3e10)
    rng = np.random.default_rng(5)
    out = {"params": {"default": {}, "custom": {
        k: (list(map(list, v)) if k == "unroll_factors" else v)
        for k, v in asdict(custom).items()
        if k not in ("noise_sigma", "noise_seed")}}, "cases": []}
    nets = [("gemm_64.yaml", TargetConfig(tiling_levels=2)),
            ("conv2d.yaml", TargetConfig()), ("bert_like.yaml", TargetConfig()),
            ("two_phase.yaml", TargetConfig()), ("gemm_l.yaml", gpu_target())]
    out["yaml"] = {}
    for wl, tg in nets:
        out["yaml"][wl] = open(os.path.join(wl_dir, wl)).read()
        net = load_network(os.path.join(wl_dir, wl))
        for sg_i, sg in enumerate(net.subgraphs[:2]):
            for k_i, sk in enumerate(generate_sketches(sg, tg)):
                ctx = SketchContext(sg, sk, tg)
                states = sample_initial_schedules(sk, 40, rng)
                rec = {"workload": wl, "target": asdict(tg), "sg": sg_i,
                       "sketch": k_i,
                       "states": [s.canonical() for s in states],
                       "default": [repr(simulate_time(s, ctx, SimHwParams()))
                                   for s in states],
                       "custom": [repr(simulate_time(s, ctx, custom))
                                  for s in states]}
                out["cases"].append(rec)
    net = load_network(os.path.join(wl_dir, "gemm_64.yaml"))
    tg = TargetConfig(tiling_levels=2)
    sg = net.subgraphs[0]
    out["brute"] = []
    for k_i, sk in enumerate(generate_sketches(sg, tg)):
        ctx = SketchContext(sg, sk, tg)
        for name, prm in (("default", SimHwParams()), ("custom", custom)):
            st, tm = brute_force_best(ctx, prm)
            out["brute"].append({"workload": "gemm_64.yaml", "sg": 0,
                                 "sketch": k_i, "target": asdict(tg),
                                 "params": name, "state": st.canonical(),
                                 "time": repr(tm)})
    path = os.path.join(HERE, "sim_golden.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)
    print("sim golden", len(out["cases"]), "cases,", len(out["brute"]),
          "brute-force optima")
    return os.path.getsize(path)


def make_gbt_fixture(n: int = 2500):
    """The reference's own GBT refit on a larger realistic training set:
    featurized uniform conv2d/GEMM states (many tied feature values) with
    SimulatedBackend throughputs, renormalized per subgraph exactly as
    training_examples() does."""
    sys.path.insert(0, REF)
    from schedtune.costmodel import GbtConfig, SurrogateModel
    from schedtune.measure import MeasureRequest, SimulatedBackend
    from schedtune.schedspace import SketchContext, sample_initial_schedules
    from schedtune.workload import TargetConfig, generate_sketches, load_network
    wl_dir = "/root/reference/pkg/workloads"
    model = SurrogateModel(GbtConfig())
    rng = np.random.default_rng(77)
    backend = SimulatedBackend()
    for wl in ("conv2d.yaml", "gemm_l.yaml"):
        net = load_network(os.path.join(wl_dir, wl))
        tg = TargetConfig()
        for sg in net.subgraphs[:2]:
            for sk in generate_sketches(sg, tg):
                ctx = SketchContext(sg, sk, tg)
                states = sample_initial_schedules(sk, n // 12, rng)
                res = backend.measure_batch([MeasureRequest(s, ctx)
                                             for s in states])
                for s_, r in zip(states, res):
                    if r.valid:
                        model.observe(ctx.featurize(s_), r.throughput, sg.id)
    ex = model.training_examples()
    X = np.stack([e.features for e in ex])
    y = np.asarray([e.target for e in ex], np.float64)
    rep = model.fit_round()
    arrays = {"X": X, "y": y, "base": np.asarray([model.base]),
              "loss": np.asarray([rep.loss_before, rep.loss_after])}
    for i, tr in enumerate(model.trees):
        arrays[f"tree{i:03d}_feature"] = tr.feature.astype(np.int16)
        arrays[f"tree{i:03d}_threshold"] = tr.threshold
        arrays[f"tree{i:03d}_left"] = tr.left.astype(np.int16)
        arrays[f"tree{i:03d}_right"] = tr.right.astype(np.int16)
        arrays[f"tree{i:03d}_value"] = tr.value
    arrays["n_trees"] = np.asarray([len(model.trees)])
    path = os.path.join(HERE, "gbt_fit_large.npz")
    np.savez_compressed(path, **arrays)
    print("gbt_fit_large", X.shape, len(model.trees), os.path.getsize(path))
    return os.path.getsize(path)


if __name__ == "__main__":
    main()
