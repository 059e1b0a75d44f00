"""ctypes binding of ``libharl_b200.so`` (declarations: include/harl_b200.h).

The library is built in-tree by ``paper_2211_11172_b200.build``.  There is
no fallback: if the library cannot be loaded, or no CUDA device is present,
every device entry point raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import DeviceError

HERE = os.path.dirname(os.path.abspath(__file__))
# HARL_LIB_PATH: a variant build (build.py --out/-D) for A/B measurements
LIB_PATH = os.environ.get("HARL_LIB_PATH") or \
    os.path.join(HERE, "libharl_b200.so")

MAX_DIMS, MAX_LEVELS, MAX_SLOTS = 16, 8, 64
MAX_STAGES, MAX_TENSORS, MAX_TERMS = 16, 48, 160
MAX_HEAD0, MAX_LAYERS, MAX_HIDDEN, MAX_FEATURES = 512, 4, 256, 128

ST_OK, ST_TILING, ST_COMPUTE_AT, ST_PARALLEL, ST_UNROLL = 0, 1, 2, 3, 4
# return codes (harl_b200.h)
E_ARG, E_CUDA, E_LIMIT = -1, -2, -3
ST_NO_VALID, ST_NONFINITE = 5, 6

i16, i32, i64, u32, u64, f64 = (C.c_int16, C.c_int32, C.c_int64, C.c_uint32,
                                C.c_uint64, C.c_double)
vp = C.c_void_p


class SketchDesc(C.Structure):
    _fields_ = [("levels", i32), ("ndims", i32), ("local_slots", i32),
                ("num_slots", i32), ("ncas", i32), ("max_fusible", i32),
                ("n_unroll", i32), ("max_feature_dims", i32),
                ("feature_len", i32), ("n_stages", i32), ("n_tensors", i32),
                ("n_terms", i32), ("max_extent", i32), ("n_head0", i32),
                ("extents", i32 * MAX_DIMS), ("tiling_counts", i32 * MAX_DIMS),
                ("tiling_offsets", i32 * MAX_DIMS),
                ("term_gi", i16 * MAX_TERMS), ("term_sc", i16 * MAX_TERMS),
                ("term_off", i16 * MAX_TERMS),
                ("tensor_first", i16 * MAX_TENSORS),
                ("tensor_nterms", i16 * MAX_TENSORS),
                ("stage_first", i16 * MAX_STAGES),
                ("stage_ntensors", i16 * MAX_STAGES),
                ("stage_inter", i16 * MAX_STAGES),
                ("stage_extra", i16 * MAX_STAGES),
                ("head0_src", i16 * MAX_HEAD0), ("head0_dst", i16 * MAX_HEAD0),
                ("flops_feature", f64), ("log2_lut", vp), ("spf_lut", vp),
                ("tiling_table", vp), ("dev_self", vp)]


class Pcg64(C.Structure):
    _fields_ = [("state_hi", u64), ("state_lo", u64), ("inc_hi", u64),
                ("inc_lo", u64), ("has_uint32", i32), ("uinteger", u32)]


class MlpDesc(C.Structure):
    _fields_ = [("n_layers", i32), ("dims", i32 * (MAX_LAYERS + 1)),
                ("W", vp * MAX_LAYERS), ("b", vp * MAX_LAYERS),
                ("head_W", vp), ("head_b", vp), ("n_head_cols", i32)]


class CopyOp(C.Structure):
    _fields_ = [("off", i64), ("flat_ld", i64), ("host", vp), ("host_ld", i64),
                ("rows", i64), ("ncols", i64), ("cols", vp)]


class ForestDesc(C.Structure):
    _fields_ = [("n_trees", i32), ("fitted", i32), ("base", f64),
                ("floor_value", f64), ("tree_first", vp), ("nodes", vp),
                ("n_nodes", i64), ("dev_hdr", vp)]


class ReplayRing(C.Structure):
    _fields_ = [("X", vp), ("Xn", vp), ("actions", vp), ("scalars", vp),
                ("move_bits", vp), ("shift_bits", vp), ("cap", i64)]


class SimDesc(C.Structure):
    _fields_ = [("cores", i32), ("n_skipped", i32), ("cap_l1", f64),
                ("cap_l2", f64), ("miss_l1", f64), ("miss_l2", f64),
                ("par_overhead", f64), ("peak_flops", f64),
                ("unroll_factor", f64 * MAX_LEVELS),
                ("stage_flops", f64 * MAX_STAGES),
                ("stage_spatial_n", i32 * MAX_STAGES),
                ("stage_spatial", (i16 * MAX_DIMS) * MAX_STAGES),
                ("skipped_flops", f64 * MAX_STAGES),
                ("skipped_l1", f64 * MAX_STAGES),
                ("skipped_l2", f64 * MAX_STAGES)]


class EntryLog(C.Structure):
    _fields_ = [("tiles", vp), ("knobs", vp), ("score", vp), ("reward", vp),
                ("track", vp), ("ld", i64)]


class TrackStats(C.Structure):
    _fields_ = [("steps", vp), ("best_score", vp), ("best_step", vp)]


class StepBuffers(C.Structure):
    _fields_ = [("row_track", vp), ("tiles_new", vp), ("knobs_new", vp),
                ("feat", vp), ("feat_new", vp), ("new_score", vp),
                ("reward", vp), ("v_cur", vp), ("v_next", vp),
                ("actions", vp), ("head0_col", vp), ("logp", vp),
                ("move_bits", vp), ("shift_bits", vp), ("adv", vp)]


class NetLayout(C.Structure):
    _fields_ = [("n_layers", i32), ("dims", i32 * (MAX_LAYERS + 1)),
                ("off_W", i64 * MAX_LAYERS), ("off_b", i64 * MAX_LAYERS),
                ("off_hW", i64), ("off_hb", i64), ("n_head_cols", i32),
                ("row_act", i32 * (MAX_LAYERS + 1)),
                ("row_delta", i32 * MAX_LAYERS), ("row_head", i32)]


class PpoHyper(C.Structure):
    _fields_ = [("clip_ratio", f64), ("entropy_weight", f64),
                ("value_loss_weight", f64), ("lr_actor", f64),
                ("lr_critic", f64), ("b1t_pi", f64), ("b2t_pi", f64),
                ("b1t_v", f64), ("b2t_v", f64), ("beta1", f64),
                ("beta2", f64), ("one_m_beta1", f64), ("one_m_beta2", f64),
                ("eps", f64)]


P = C.POINTER
_SIGS = {
    "harl_abi_version": (i32, []),
    "harl_prepare": (i32, []),
    "harl_last_error": (C.c_char_p, []),
    "harl_device_query": (i32, [i32, P(i32), P(i32), P(i32)]),
    "harl_init_population": (i32, [P(SketchDesc), P(Pcg64), i64, vp, vp, i64,
                                   P(i64), vp, vp]),
    "harl_rng_prepare": (i32, [P(Pcg64)]),
    "harl_featurize": (i32, [P(SketchDesc), vp, vp, i64, i64, vp, vp]),
    "harl_uniform_scratch_bytes": (i64, [i64]),
    "harl_uniform_actions": (i32, [P(SketchDesc), vp, vp, i64, i64, P(Pcg64),
                                   vp, vp, P(i64), vp]),
    "harl_action_masks": (i32, [P(SketchDesc), vp, vp, i64, i64, vp, vp, vp]),
    "harl_apply_actions": (i32, [P(SketchDesc), vp, vp, i64, i64, vp, vp, vp,
                                 vp, vp]),
    "harl_gbt_predict": (i32, [P(ForestDesc), vp, i64, i32, vp, vp, vp, vp]),
    "harl_policy_step": (i32, [P(SketchDesc), P(MlpDesc), vp, vp, vp, i64, i64,
                               P(Pcg64), vp, vp, vp, vp, vp, vp, vp, vp, vp,
                               vp, vp, i64, vp]),
    "harl_value_forward": (i32, [P(MlpDesc), vp, i64, i32, vp, vp]),
    "harl_policy_step_tc": (i32, [P(SketchDesc), P(MlpDesc), vp, vp, vp, i64,
                                  i64, P(Pcg64), vp, vp, vp, vp, vp, vp, vp,
                                  vp, vp, vp, vp, vp, vp, vp, vp, i64, vp,
                                  i32, vp]),
    "harl_policy_step_tc_gbt": (i32, [P(SketchDesc), P(MlpDesc), vp, vp, vp,
                                      i64, i64, P(Pcg64), vp, vp, vp, vp, vp,
                                      vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                      i64, vp, i32, P(ForestDesc), vp, vp, vp,
                                      vp]),
    "harl_value_pair_tc": (i32, [P(MlpDesc), vp, i64, vp, i64, i32, vp, vp,
                                 vp, i32, vp]),
    "harl_value_finish_tc": (i32, [P(MlpDesc), vp, i64, vp, i64, i32, vp, vp,
                                   vp, i32, P(StepBuffers), i64, i64, i32,
                                   f64, i32, P(ReplayRing), i64, i64,
                                   P(EntryLog), P(TrackStats), vp, vp]),
    "harl_tc_packed_bytes": (i64, [i32, i32]),
    "harl_pack_tc_weights": (i32, [P(MlpDesc), P(MlpDesc), i32, vp, vp, vp,
                                   vp]),
    "harl_finish_step": (i32, [P(StepBuffers), i64, i64, i64, i32, i32, f64,
                               i32, P(ReplayRing), i64, i64, P(EntryLog),
                               P(TrackStats), vp, vp]),
    "harl_gbt_finish_step": (i32, [P(ForestDesc), i32, vp, P(StepBuffers), i64,
                                   i64, i64, i32, f64, i32, P(ReplayRing),
                                   i64, i64, P(EntryLog), P(TrackStats), vp,
                                   vp]),
    "harl_gather_rows": (i32, [vp, i64, i32, i32, vp, vp, vp, vp, vp, i64, vp,
                               vp, vp, vp, vp, i64, vp]),
    "harl_ppo_scratch_bytes": (i64, [i32, i32, i32]),
    "harl_rank_scratch_bytes": (i64, [i64, i64]),
    "harl_sim_time": (i32, [P(SketchDesc), P(SimDesc), vp, vp, i64, i64, vp,
                            vp]),
    "harl_brute_force": (i32, [P(SketchDesc), P(SimDesc), u64, u64, vp, vp,
                               vp, i64, vp]),
    "harl_heap_to_creation_order": (i32, [vp, vp, vp, i32, i32, vp, vp, vp,
                                          vp, vp, vp]),
    "harl_format_floats": (C.c_longlong, [vp, C.c_longlong, vp, C.c_longlong,
                                          i32]),
    "harl_format_canonical": (C.c_longlong, [vp, vp, C.c_longlong, i32, i32,
                                              C.c_char_p, C.c_longlong, vp,
                                              C.c_longlong]),
    "harl_agent_copy": (i32, [P(CopyOp), i32, vp, i32]),
    "harl_forest_pack": (C.c_longlong, [i32, vp, vp, vp, vp, vp, vp, f64, vp,
                                         vp, i32, vp, C.c_longlong,
                                         P(C.c_longlong)]),
    "harl_cull_select": (i32, [vp, vp, i64, vp, i64, i64, vp, vp, P(i64)]),
    "harl_gbt_fit_scratch_bytes": (i64, [i32, i32, i32]),
    "harl_gbt_fit": (i32, [vp, vp, i32, i32, i32, i32, f64, i32, vp, i64, vp,
                           vp, vp, vp, vp, vp, vp, vp]),
    "harl_rank_topk": (i32, [P(EntryLog), i32, i64, vp, vp, i64, i64, i64,
                             vp, i64, vp, i64, vp, vp]),
    "harl_selftest_tcgen05": (i32, [vp, vp, vp, i32, vp]),
    "harl_launch_count": (C.c_longlong, []),
    "harl_debug_timestamps": (i32, [i32, vp, i32]),
    "harl_profile_set": (i32, [i32, C.c_longlong]),
    "harl_profile_reset": (i32, []),
    "harl_profile_read": (i32, [i32, C.c_char_p, i32, vp, vp, vp]),
    "harl_ppo_update": (i32, [P(NetLayout), P(NetLayout), P(PpoHyper),
                              P(ReplayRing), vp, i32, i32, i32, vp, i32, vp,
                              vp, vp, vp, vp, i64, i64, vp, vp, vp, vp, vp,
                              vp, vp, vp, i32, i32, vp]),
    "harl_ppo_wt_doubles": (i64, [P(NetLayout), P(NetLayout)]),
    "harl_ppo_wt_fill": (i32, [P(NetLayout), P(NetLayout), vp, vp, vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_device_ok = False     # a CUDA device was seen (checked once, not per call)


def load(require_device: bool = True):
    """Load (once) and return the ctypes library.

    ``require_device=False`` only checks that the shared object loads and
    exports every symbol (used by the CPU test suite)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"native library missing: {LIB_PATH} (run "
                "`python -m paper_2211_11172_b200.build`)")
        try:
            lib = C.CDLL(LIB_PATH)
        except OSError as exc:
            raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.harl_abi_version() != 1:
            raise DeviceError("ABI version mismatch")
        _lib = lib
    if require_device and not _device_ok:
        import torch
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device: the B200 path has no CPU "
                              "fallback")
        globals()["_device_ok"] = True
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = _lib.harl_last_error().decode() if _lib is not None else ""
        raise DeviceError(f"{what} failed ({rc}): {msg}")
