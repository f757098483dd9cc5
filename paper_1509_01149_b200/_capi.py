"""ctypes mirror of include/mppi.h (argument marshalling only).

Loads the in-tree libmppi_b200.so.  There is no fallback: if the library is missing
or cannot be loaded the import fails loudly.
"""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MPPI_LIB: an alternative in-tree build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("MPPI_LIB") or os.path.join(HERE, "libmppi_b200.so")

MPPI_OK, MPPI_ERR_INVALID_ARG, MPPI_ERR_NOT_SPD, MPPI_ERR_OOM, MPPI_ERR_CUDA, MPPI_ERR_UNSUPPORTED = \
    0, 1, 2, 3, 4, 6
MPPI_ERR_NCCL = 5
MPPI_NCCL_ID_BYTES = 128
MPPI_PLANT_CARTPOLE, MPPI_PLANT_RACECAR, MPPI_PLANT_QUADROTOR, MPPI_PLANT_LINEAR = 1, 2, 3, 4
MPPI_MAX_OBSTACLES = 4096
MPPI_OPTION_CUDA_GRAPH, MPPI_OPTION_PACKED_SAMPLES, MPPI_OPTION_FUSED_NOISE, MPPI_OPTION_OBSTACLE_GRID = \
    1, 2, 3, 4
MPPI_OPTION_BULK_REDUCTION = 5
MPPI_OPTION_PDL = 6
MPPI_OPTION_SPARSE_REDUCTION = 7
MPPI_OPTION_FUSED_REDUCTION = 8
MPPI_OPTION_GATHER_COMBINE = 9
MPPI_OPTION_NOISE_AHEAD = 10
MPPI_WEIGHTS_TRAJECTORY, MPPI_WEIGHTS_COST_TO_GO = 0, 1


class cartpole_dynamics_t(C.Structure):
    _fields_ = [("g", C.c_float), ("pole_length", C.c_float), ("vel_gain", C.c_float)]


class racecar_dynamics_t(C.Structure):
    _fields_ = [(n, C.c_float) for n in (
        "mass", "Iz", "lf", "lr", "tire_B", "tire_C", "mu", "Cm", "Cr", "Cd", "v_min", "g",
        "steer_max", "throttle_min", "throttle_max")]


class quadrotor_dynamics_t(C.Structure):
    _fields_ = [(n, C.c_float) for n in (
        "mass", "arm", "Ixx", "Iyy", "Izz", "yaw_coeff", "motor_gain", "g", "thrust_min",
        "thrust_max", "cos_phi_min")]


class linear_dynamics_t(C.Structure):
    _fields_ = [("n", C.c_int32), ("A", C.c_float * 64), ("B", C.c_float * 32)]


class _dyn_union(C.Union):
    _fields_ = [("cartpole", cartpole_dynamics_t), ("racecar", racecar_dynamics_t),
                ("quadrotor", quadrotor_dynamics_t), ("linear", linear_dynamics_t)]


class dynamics_t(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("plant", C.c_int32), ("p", _dyn_union)]


class cartpole_cost_t(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("w_p", "w_theta", "w_thetadot", "w_pdot")]


class racecar_cost_t(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("track_a", "track_b", "w_track", "w_speed", "v_ref")]


class quadrotor_cost_t(C.Structure):
    _fields_ = [("goal", C.c_float * 3)] + [(n, C.c_float) for n in (
        "w_xy", "w_z", "w_yaw", "w_vel", "w_obs", "obs_length", "w_crash", "ground_z",
        "obstacle_radius")] + [("n_obstacles", C.c_int32), ("obstacles_xy", C.POINTER(C.c_float))]


class linear_cost_t(C.Structure):
    _fields_ = [("Q", C.c_float * 64)]


class _cost_union(C.Union):
    _fields_ = [("cartpole", cartpole_cost_t), ("racecar", racecar_cost_t),
                ("quadrotor", quadrotor_cost_t), ("linear", linear_cost_t)]


class cost_t(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("penalty", C.c_float), ("p", _cost_union)]


class dist_t(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32)]


class info_t(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("T", C.c_int32), ("plant", C.c_int32),
                ("K", C.c_int64), ("K_loc", C.c_int64), ("k_offset", C.c_int64),
                ("n_chunks", C.c_int32), ("reserved", C.c_int32), ("workspace_bytes", C.c_size_t)]


class stats_t(C.Structure):
    _fields_ = [("k_star", C.c_int64), ("s_min", C.c_float), ("eta", C.c_float)]


class kernel_times_t(C.Structure):
    _fields_ = [("total_ms", C.c_double * 6), ("launches", C.c_int64 * 6)]


KERNEL_NAMES = ["noise", "rollout", "wsum", "finalize", "shift", "collective"]

EXPORTS = ["mppi_create", "mppi_destroy", "mppi_info", "mppi_set_stream", "mppi_optimize", "mppi_use_graph", "mppi_set_option",
           "mppi_optimize_host", "mppi_rollout_costs", "mppi_accumulate", "mppi_gather_record_len", "mppi_accumulate_record", "mppi_apply_gathered", "mppi_apply",
           "mppi_shift", "mppi_noise", "mppi_feynman_kac", "mppi_closed_loop", "mppi_set_weighting",
           "mppi_cost_to_go", "mppi_set_sampling_transform", "mppi_nccl_unique_id", "mppi_nccl_attach",
           "mppi_obstacle_grid", "mppi_plant_step", "mppi_get_stats", "mppi_replay_count",
           "mppi_last_launch_count", "mppi_last_kernels", "mppi_profile_enable", "mppi_profile_read", "mppi_last_error", "mppi_status_string", "mppi_abi_version"]

_lib = None


def lib():
    """The loaded libmppi_b200.so (raises if absent: there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError("libmppi_b200.so not built (%s); run python -m paper_1509_01149_b200.build "
                          "or __graft_entry__.build()" % LIB_PATH)
    L = C.CDLL(LIB_PATH)
    vp, fp, dp = C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_double)
    i64p = C.POINTER(C.c_int64)
    st = C.c_int
    L.mppi_create.argtypes = [C.POINTER(dynamics_t), C.POINTER(cost_t), C.c_int64, C.c_int32,
                              C.c_float, C.c_float, C.c_float, C.c_int32, dp, dp,
                              C.POINTER(dist_t), vp, C.POINTER(vp)]
    L.mppi_create.restype = st
    L.mppi_destroy.argtypes = [vp]
    L.mppi_destroy.restype = None
    L.mppi_info.argtypes = [vp, C.POINTER(info_t)]
    L.mppi_info.restype = st
    L.mppi_set_stream.argtypes = [vp, vp]
    L.mppi_set_stream.restype = st
    L.mppi_optimize.argtypes = [vp, fp, vp, C.c_uint64, C.c_uint64, vp]
    L.mppi_optimize.restype = st
    L.mppi_set_option.argtypes = [vp, C.c_int, C.c_int32]
    L.mppi_set_option.restype = st
    L.mppi_use_graph.argtypes = [vp, C.c_int32]
    L.mppi_use_graph.restype = st
    L.mppi_optimize_host.argtypes = [vp, fp, fp, C.c_uint64, C.c_uint64]
    L.mppi_optimize_host.restype = st
    L.mppi_rollout_costs.argtypes = [vp, fp, vp, C.c_uint64, C.c_uint64, vp, vp, vp]
    L.mppi_rollout_costs.restype = st
    L.mppi_accumulate.argtypes = [vp, vp, vp]
    L.mppi_accumulate.restype = st
    L.mppi_apply.argtypes = [vp, vp, vp]
    L.mppi_apply.restype = st
    L.mppi_gather_record_len.argtypes = [vp]
    L.mppi_gather_record_len.restype = C.c_int64
    L.mppi_accumulate_record.argtypes = [vp, vp]
    L.mppi_accumulate_record.restype = st
    L.mppi_apply_gathered.argtypes = [vp, vp, vp, C.c_int32]
    L.mppi_apply_gathered.restype = st
    L.mppi_shift.argtypes = [vp, vp, fp]
    L.mppi_shift.restype = st
    L.mppi_obstacle_grid.argtypes = [C.POINTER(C.c_float), C.c_int32, C.POINTER(C.c_uint32), C.c_int64,
                                     C.POINTER(C.c_float)]
    L.mppi_obstacle_grid.restype = st
    L.mppi_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8)]
    L.mppi_nccl_unique_id.restype = st
    L.mppi_nccl_attach.argtypes = [vp, C.POINTER(C.c_uint8)]
    L.mppi_nccl_attach.restype = st
    L.mppi_set_sampling_transform.argtypes = [vp, dp]
    L.mppi_set_sampling_transform.restype = st
    L.mppi_set_weighting.argtypes = [vp, C.c_int]
    L.mppi_set_weighting.restype = st
    L.mppi_cost_to_go.argtypes = [vp, vp]
    L.mppi_cost_to_go.restype = st
    L.mppi_closed_loop.argtypes = [vp, vp, vp, C.c_uint64, C.c_uint64, C.c_int32, fp, C.c_int32, vp, vp, vp]
    L.mppi_closed_loop.restype = st
    L.mppi_feynman_kac.argtypes = [vp, fp, C.c_uint64, C.c_uint64, dp]
    L.mppi_feynman_kac.restype = st
    L.mppi_noise.argtypes = [vp, C.c_uint64, C.c_uint64, vp]
    L.mppi_noise.restype = st
    L.mppi_plant_step.argtypes = [vp, fp, fp, C.POINTER(C.c_int32), fp]
    L.mppi_plant_step.restype = st
    L.mppi_get_stats.argtypes = [vp, C.POINTER(stats_t)]
    L.mppi_get_stats.restype = st
    L.mppi_replay_count.argtypes = [vp, C.POINTER(C.c_int64)]
    L.mppi_replay_count.restype = st
    L.mppi_last_launch_count.argtypes = [vp]
    L.mppi_last_launch_count.restype = C.c_int32
    L.mppi_last_kernels.argtypes = [vp, C.c_char_p, C.c_int64]
    L.mppi_last_kernels.restype = C.c_int64
    L.mppi_profile_enable.argtypes = [vp, C.c_int32]
    L.mppi_profile_enable.restype = st
    L.mppi_profile_read.argtypes = [vp, C.POINTER(kernel_times_t)]
    L.mppi_profile_read.restype = st
    L.mppi_last_error.argtypes = []
    L.mppi_last_error.restype = C.c_char_p
    L.mppi_status_string.argtypes = [C.c_int]
    L.mppi_status_string.restype = C.c_char_p
    L.mppi_abi_version.argtypes = []
    L.mppi_abi_version.restype = C.c_int32
    _lib = L
    return L


class MppiError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (lib().mppi_status_string(status).decode(), msg))
        self.status = status


def check(status):
    if status != MPPI_OK:
        raise MppiError(status, lib().mppi_last_error().decode())
    return status
