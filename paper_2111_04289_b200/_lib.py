"""ctypes binding of liblmstream.so (include/lmstream.h) — argument marshalling only.

Every function here has the C name and forwards to the shared library; there is no
Python fallback: importing this module on a machine without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblmstream.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python paper_2111_04289_b200/build.py` "
                      "(the LMStream hot path has no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

# ---------------------------------------------------------------- constants
LMS_ABI_VERSION = 3
LMS_OK, LMS_EINVAL, LMS_ENOMEM, LMS_ECUDA, LMS_ENCCL, LMS_EHISTORY, LMS_EPLAN, LMS_EFORMAT, \
    LMS_ESTATE, LMS_EOVERFLOW, LMS_EINTERNAL = 0, -1, -2, -3, -4, -5, -6, -7, -8, -9, -10
STATUS_NAMES = {0: "LMS_OK", -1: "LMS_EINVAL", -2: "LMS_ENOMEM", -3: "LMS_ECUDA", -4: "LMS_ENCCL",
                -5: "LMS_EHISTORY", -6: "LMS_EPLAN", -7: "LMS_EFORMAT", -8: "LMS_ESTATE",
                -9: "LMS_EOVERFLOW", -10: "LMS_EINTERNAL"}
LMS_LR1S, LMS_LR1T, LMS_LR2S, LMS_CM1S, LMS_CM1T, LMS_CM2S = range(6)
KIND = {"LR1S": 0, "LR1T": 1, "LR2S": 2, "CM1S": 3, "CM1T": 4, "CM2S": 5}
LMS_MODE_LMSTREAM, LMS_MODE_DEADLINE, LMS_MODE_TRIGGER, LMS_MODE_MANUAL = range(4)
MODE = {"lmstream": 0, "deadline": 1, "trigger": 2, "manual": 3}
LMS_FLAG_ONLINE_INFPT = 1
LMS_FLAG_PIPELINE = 2
LMS_FLAG_DENSE_VEHICLES = 4
LMS_FLAG_NVLS = 8
LMS_OP_SCAN, LMS_OP_FILTER, LMS_OP_PROJECT, LMS_OP_HASHAGG, LMS_OP_HASHJOIN, LMS_OP_SORT, \
    LMS_OP_SHUFFLE, LMS_OP_EXPAND = range(8)
LMS_DEV_CPU, LMS_DEV_GPU = 0, 1
ADMIT_REASONS = {0: "forced", 1: "bootstrap", 2: "target", 3: "tumbling-bootstrap", 4: "cap",
                 5: "trigger", 6: "flush", -1: "buffer", -2: "poll"}


# ---------------------------------------------------------------- structs
class lms_config(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("kind", C.c_int32), ("mode", C.c_int32),
                ("device", C.c_int32), ("deadline_s", C.c_double), ("trigger_s", C.c_double),
                ("range_s", C.c_double), ("slide_s", C.c_double), ("num_cores", C.c_int32),
                ("num_xways", C.c_int32), ("inf_pt_bytes", C.c_double), ("base_trans_cost", C.c_double),
                ("max_batch_bytes", C.c_uint64), ("max_keys", C.c_uint64), ("max_result_rows", C.c_uint64),
                ("pane_slots", C.c_uint32), ("flags", C.c_uint32), ("rank", C.c_int32), ("world", C.c_int32),
                ("num_gpus", C.c_int32), ("device_ids", C.POINTER(C.c_int32))]


class lms_agg_row(C.Structure):
    _fields_ = [("win_start_s", C.c_int64), ("win_end_s", C.c_int64), ("key", C.c_uint64),
                ("count", C.c_uint64), ("sum_fixed", C.c_uint64), ("sum", C.c_double), ("avg", C.c_double),
                ("key_xway", C.c_uint32), ("key_dir", C.c_uint32), ("key_seg", C.c_uint32),
                ("rank", C.c_uint32)]


class lms_lr1_row(C.Structure):
    _fields_ = [("win_start_s", C.c_int64), ("vehicle", C.c_uint64), ("ts", C.c_uint32),
                ("multiplicity", C.c_uint32), ("speed", C.c_uint16), ("xway", C.c_uint16),
                ("segment", C.c_uint16), ("lane", C.c_uint8), ("dir", C.c_uint8)]


class lms_batch_record(C.Structure):
    _fields_ = [("index", C.c_uint64), ("num_datasets", C.c_uint64), ("num_records", C.c_uint64),
                ("batch_bytes", C.c_uint64), ("admit_time_s", C.c_double), ("max_buff_s", C.c_double),
                ("proc_s", C.c_double), ("device_s", C.c_double), ("h2d_s", C.c_double),
                ("d2h_s", C.c_double), ("max_lat_s", C.c_double), ("est_max_lat_s", C.c_double),
                ("avg_thput_Bps", C.c_double), ("inf_pt_bytes", C.c_double), ("n_cpu_ops", C.c_uint32),
                ("n_gpu_ops", C.c_uint32), ("plan_mask", C.c_uint32), ("admit_reason", C.c_uint32),
                ("plan_overhead_s", C.c_double), ("admit_overhead_s", C.c_double),
                ("windows_closed", C.c_uint64), ("rows_emitted", C.c_uint64), ("late_records", C.c_uint64),
                ("bad_records", C.c_uint64), ("overflow_records", C.c_uint64), ("watermark", C.c_int64),
                ("opt_overhead_s", C.c_double), ("opt_block_s", C.c_double)]


class lms_p2p_handle(C.Structure):
    _fields_ = [("rank", C.c_uint32), ("world", C.c_uint32), ("K", C.c_uint32), ("kind", C.c_uint32),
                ("dict_cap_mask", C.c_uint64), ("dict_max_keys", C.c_uint32), ("present", C.c_uint32),
                ("ipc", (C.c_uint8 * 64) * 6)]


class lms_dag(C.Structure):
    _fields_ = [("n", C.c_uint32), ("op_kind", C.POINTER(C.c_uint8)), ("pred_off", C.POINTER(C.c_int32)),
                ("preds", C.POINTER(C.c_int32))]


assert C.sizeof(lms_agg_row) == 72 and C.sizeof(lms_lr1_row) == 32

# ---------------------------------------------------------------- prototypes
_P = C.POINTER
_Q = C.c_void_p
_PROTOS = {
    "lms_abi_version": (C.c_uint32, []),
    "lms_last_error": (C.c_char_p, []),
    "lms_config_init": (C.c_int32, [_P(lms_config), C.c_int32]),
    "lms_query_create": (C.c_int32, [_P(lms_config), _P(_Q)]),
    "lms_query_destroy": (C.c_int32, [_Q]),
    "lms_push": (C.c_int32, [_Q, C.c_void_p, C.c_uint64, C.c_double, _P(C.c_uint64)]),
    "lms_push_pinned": (C.c_int32, [_Q, C.c_void_p, C.c_uint64, C.c_double, _P(C.c_uint64)]),
    "lms_push_device": (C.c_int32, [_Q, C.c_void_p, C.c_uint64, C.c_double, _P(C.c_uint64)]),
    "lms_poll": (C.c_int32, [_Q, C.c_double, _P(C.c_int32), _P(C.c_uint64)]),
    "lms_force_batch": (C.c_int32, [_Q, C.c_double, _P(C.c_uint64)]),
    "lms_flush": (C.c_int32, [_Q, C.c_double]),
    "lms_sync": (C.c_int32, [_Q]),
    "lms_read_agg": (C.c_int32, [_Q, _P(lms_agg_row), C.c_uint64, _P(C.c_uint64), _P(C.c_uint64)]),
    "lms_read_lr1": (C.c_int32, [_Q, _P(lms_lr1_row), C.c_uint64, _P(C.c_uint64), _P(C.c_uint64)]),
    "lms_num_batches": (C.c_int32, [_Q, _P(C.c_uint64)]),
    "lms_get_batch_record": (C.c_int32, [_Q, C.c_uint64, _P(lms_batch_record)]),
    "lms_watermark_ptrs": (C.c_int32, [_Q, _P(C.c_void_p), _P(C.c_void_p), _P(C.c_void_p)]),
    "lms_run_close": (C.c_int32, [_Q]),
    "lms_partials": (C.c_int32, [_Q, _P(C.c_void_p), _P(C.c_uint64)]),
    "lms_merge": (C.c_int32, [_Q, C.c_void_p, C.c_uint64]),
    "lms_close_range": (C.c_int32, [_Q, _P(C.c_int64), _P(C.c_int64)]),
    "lms_lr1_window_counts": (C.c_int32, [_Q, C.c_int64, _P(C.c_void_p), _P(C.c_uint64)]),
    "lms_lr1_probe": (C.c_int32, [_Q, C.c_int64]),
    "lms_p2p_export": (C.c_int32, [_Q, _P(lms_p2p_handle)]),
    "lms_p2p_import": (C.c_int32, [_Q, _P(lms_p2p_handle)]),
    "lms_p2p_import_local": (C.c_int32, [_Q, _Q]),
    "lms_merge_window": (C.c_int32, [_Q, _P(C.c_uint32)]),
    "lms_last_close_range": (C.c_int32, [_Q, _P(C.c_int64), _P(C.c_int64)]),
    "lms_p2p_push": (C.c_int32, [_Q, C.c_int64, C.c_uint32]),
    "lms_p2p_finalize": (C.c_int32, [_Q, C.c_int64, C.c_uint32]),
    "lms_p2p_exchange_async": (C.c_int32, [_Q]),
    "lms_p2p_collect": (C.c_int32, [_Q]),
    "lms_p2p_device_watermark": (C.c_int32, [_Q, C.c_int32]),
    "lms_nvls_active": (C.c_int32, [_Q, _P(C.c_int32)]),
    "lms_dense_partials": (C.c_int32, [_Q, C.c_int64, C.c_uint32, _P(C.c_void_p), _P(C.c_void_p), _P(C.c_uint64)]),
    "lms_dense_finalize": (C.c_int32, [_Q, C.c_int64, C.c_uint32]),
    "lms_split": (C.c_int32, [C.c_int32, C.c_void_p, C.c_uint64, C.c_uint32, _P(C.c_uint64)]),
    "lms_last_kernel_times": (C.c_int32, [_Q, _P(C.c_double), _P(C.c_double), _P(C.c_double)]),
    "lms_kernel_launches": (C.c_int32, [_Q, _P(C.c_uint64)]),
    "lms_est_max_lat": (C.c_int32, [_P(C.c_double), _P(C.c_uint64), C.c_uint64, C.c_double, _P(C.c_double)]),
    "lms_cpu_cost": (C.c_int32, [C.c_double, C.c_double, C.c_double, _P(C.c_double)]),
    "lms_gpu_cost": (C.c_int32, [C.c_double, C.c_double, C.c_double, _P(C.c_double)]),
    "lms_trans_cost": (C.c_int32, [C.c_double, C.c_double, C.c_double, _P(C.c_double)]),
    "lms_base_cost": (C.c_int32, [C.c_int32, _P(C.c_double)]),
    "lms_map_device": (C.c_int32, [_P(lms_dag), C.c_double, C.c_double, C.c_double, _P(C.c_uint8)]),
    "lms_query_dag": (C.c_int32, [C.c_int32, _P(lms_dag)]),
    "lms_admit_decision": (C.c_int32, [C.c_int32, C.c_double, C.c_double, C.c_double, _P(C.c_double),
                                       _P(C.c_uint64), C.c_uint64, C.c_double, _P(C.c_double), C.c_uint64,
                                       _P(C.c_int32), _P(C.c_double), _P(C.c_int32)]),
    "lms_infpt_fit": (C.c_int32, [_P(C.c_double), _P(C.c_double), _P(C.c_double), C.c_uint64,
                                  _P(C.c_double), _P(C.c_double), _P(C.c_double)]),
    "lms_infpt_predict": (C.c_int32, [C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                      _P(C.c_double)]),
    "lms_percentile": (C.c_int32, [_P(C.c_double), C.c_uint64, C.c_double, _P(C.c_double)]),
}
for _name, (_res, _args) in _PROTOS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f

EXPORTED = tuple(_PROTOS)


class LmsError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = lms_last_error()
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {msg.decode() if msg else ''}")


def check(status: int, where: str = "lms", ok=(LMS_OK,)) -> int:
    if status not in ok:
        raise LmsError(status, where)
    return status
