"""ctypes binding of the C-ABI in include/pact_cuda.h.

This is the Python view of the drop-in boundary: the same entry points the C++
host API (paper_2409_10876_b200/include/pact/*.hpp) calls.  Device buffers are
passed as raw pointers (torch CUDA tensors' data_ptr(), or pact_device_alloc).
There is no fallback: if libpact_cuda.so is missing the import fails.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PACT_LIB") or os.path.join(_HERE, "lib", "libpact_cuda.so")

PACT_OK = 0
PACT_E_VALIDATION = 2
PACT_E_NUMERICAL = 3
PACT_E_CUDA = 4
PACT_E_UNSUPPORTED = 5


class PactError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[pact {code}] {msg}")
        self.code = code


class ValidationError(PactError):
    """The reference's pact::ValidationError (core.hpp:35-38)."""


class NumericalError(PactError):
    """The reference's pact::NumericalError (core.hpp:41-44)."""


class Ring(C.Structure):
    _fields_ = [("n_transducers", C.c_int32), ("radius", C.c_double),
                ("angle_offset", C.c_double)]


class Grid(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("pitch", C.c_double),
                ("origin_x", C.c_double), ("origin_y", C.c_double)]


class SignalMeta(C.Structure):
    _fields_ = [("n_samples", C.c_int32), ("dt", C.c_double), ("t0", C.c_double),
                ("background_sos", C.c_double)]


class Mask(C.Structure):
    _fields_ = [("center_x", C.c_double), ("center_y", C.c_double), ("radius", C.c_double)]


class Partition(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32)]


class Body(C.Structure):
    _fields_ = [("center_x", C.c_double), ("center_y", C.c_double), ("radius", C.c_double),
                ("body_sos", C.c_double)]


class Layout(C.Structure):
    _fields_ = [("grid", Grid), ("patch_pixels", C.c_int32), ("stride_pixels", C.c_int32),
                ("nx", C.c_int32), ("ny", C.c_int32), ("last_x", C.c_int32),
                ("last_y", C.c_int32)]


class Siren(C.Structure):
    _fields_ = [("in_dim", C.c_int32), ("hidden", C.c_int32), ("n_hidden_layers", C.c_int32),
                ("omega0", C.c_double), ("out_scale", C.c_double), ("v0", C.c_double)]


class DeconvOptions(C.Structure):
    _fields_ = [("eps", C.c_double), ("n_angles", C.c_int32), ("ray_step", C.c_double),
                ("merge_fwhm", C.c_double)]


class TrainConfig(C.Structure):
    _fields_ = [("epochs", C.c_int32), ("steps_per_epoch", C.c_int32),
                ("learning_rate", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("adam_eps", C.c_double), ("lambda_tv", C.c_double), ("n_delays", C.c_int32),
                ("delays", C.POINTER(C.c_double)), ("eps_deconv", C.c_double),
                ("n_angles", C.c_int32), ("ray_step", C.c_double), ("seed", C.c_uint64),
                ("hidden", C.c_int32), ("sine_layers", C.c_int32), ("omega0", C.c_double),
                ("out_scale", C.c_double), ("patch_mm", C.c_double), ("overlap", C.c_double),
                ("merge_fwhm", C.c_double), ("implicit_xhat_grad", C.c_int32),
                ("workers", C.c_int32), ("use_cuda_graph", C.c_int32)]


_P = C.c_void_p
_D = C.c_double
_I = C.c_int32
_DP = C.POINTER(C.c_double)
_IP = C.POINTER(C.c_int32)
_FP = C.POINTER(C.c_float)

# name -> (restype, argtypes); every symbol declared in include/pact_cuda.h.
SIGNATURES = {
    "pact_abi_version": (C.c_int, []),
    "pact_last_error": (C.c_char_p, []),
    "pact_ctx_last_error": (C.c_char_p, [C.c_void_p]),
    "pact_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "pact_ctx_destroy": (C.c_int, [_P]),
    "pact_ctx_stream": (_P, [_P]),
    "pact_ctx_set_stream": (C.c_int, [_P, _P]),
    "pact_ctx_use_own_stream": (C.c_int, [_P]),
    "pact_ctx_synchronize": (C.c_int, [_P]),
    "pact_ctx_launch_count": (C.c_int64, [_P]),
    "pact_device_alloc": (C.c_int, [_P, C.c_size_t, C.POINTER(_P)]),
    "pact_device_free": (C.c_int, [_P, _P]),
    "pact_host_alloc_pinned": (C.c_int, [C.c_size_t, C.POINTER(_P)]),
    "pact_host_free_pinned": (C.c_int, [_P]),
    "pact_upload": (C.c_int, [_P, _P, _P, C.c_size_t]),
    "pact_download": (C.c_int, [_P, _P, _P, C.c_size_t]),
    "pact_memset": (C.c_int, [_P, _P, C.c_int, C.c_size_t]),
    "pact_make_delays": (C.c_int, [_D, _D, _I, _DP]),
    "pact_das_stack": (C.c_int, [_P, C.POINTER(Ring), C.POINTER(SignalMeta), _P,
                                 C.POINTER(Grid), _D, _DP, _I, _P]),
    "pact_psnr": (C.c_int, [_P, _P, _P, _I, _I, _D, _DP]),
    "pact_ssim": (C.c_int, [_P, _P, _P, _I, _I, _D, _DP]),
    "pact_sos_rmse_masked": (C.c_int, [_P, _P, _P, C.POINTER(Grid), C.POINTER(Mask), _DP]),
    "pact_dual_sos_das": (C.c_int, [_P, C.POINTER(Ring), C.POINTER(SignalMeta), _P,
                                    C.POINTER(Grid), _D, C.POINTER(Body), _P]),
    "pact_simulate_signals": (C.c_int, [_P, C.POINTER(Grid), _DP, _DP, C.POINTER(Mask), _D,
                                        C.POINTER(Ring), _D, C.POINTER(SignalMeta), _D, _P]),
    "pact_simulate_signals_ex": (C.c_int, [_P, C.POINTER(Grid), _DP, _DP, C.POINTER(Mask), _D,
                                           C.POINTER(Ring), _D, C.POINTER(SignalMeta), _D,
                                           C.c_int32, _P]),
    "pact_simulate_window": (C.c_int, [C.POINTER(Grid), _DP, _DP, _D, C.POINTER(Ring), _D, _D, _D,
                                       C.c_int32, C.POINTER(SignalMeta)]),
    "pact_make_patch_layout": (C.c_int, [C.POINTER(Grid), _D, _D, C.POINTER(Layout)]),
    "pact_layout_n_patches": (C.c_int32, [C.POINTER(Layout)]),
    "pact_layout_patches": (C.c_int, [C.POINTER(Layout), _IP, _DP]),
    "pact_siren_param_count": (C.c_int64, [C.POINTER(Siren)]),
    "pact_init_siren": (C.c_int, [C.c_uint64, C.POINTER(Siren), _DP]),
    "pact_masked_count": (C.c_int32, [C.POINTER(Grid), C.POINTER(Mask)]),
    "pact_masked_pixels": (C.c_int, [C.POINTER(Grid), C.POINTER(Mask), _IP, _FP]),
    "pact_render_sos": (C.c_int, [_P, C.POINTER(Siren), _P, C.POINTER(Grid), C.POINTER(Mask),
                                  _P, _P]),
    "pact_siren_backward": (C.c_int, [_P, C.POINTER(Siren), _P, C.POINTER(Grid),
                                      C.POINTER(Mask), _P, _P]),
    "pact_wavefront": (C.c_int, [_P, C.POINTER(Ring), C.POINTER(Grid), _P, _D, C.POINTER(Mask),
                                 _I, _DP, _I, _D, _P]),
    "pact_transfer_stack": (C.c_int, [_P, _I, _P, _I, _DP, _I, _I, _D, _P]),
    "pact_patch_spectra": (C.c_int, [_P, C.POINTER(Layout), _P, _I, _P]),
    "pact_deconvolve_image": (C.c_int, [_P, _P, _I, _DP, _D, _P, C.POINTER(Ring),
                                        C.POINTER(Mask), C.POINTER(Layout),
                                        C.POINTER(DeconvOptions), _P]),
    "pact_loss_grad": (C.c_int, [_P, _I, _P, _P, _I, _DP, _I, _I, _D, _D, _D, _I, _P, _P]),
    "pact_ray_backward": (C.c_int, [_P, C.POINTER(Ring), C.POINTER(Grid), _P, _D,
                                    C.POINTER(Mask), _I, _DP, _I, _D, _P, _P]),
    "pact_tv_loss": (C.c_int, [_P, C.POINTER(Grid), C.POINTER(Mask), _P, _D, _DP, _P]),
    "pact_merge_window": (C.c_int, [_D, _I, _D, _DP]),
    "pact_merge_patches": (C.c_int, [_P, C.POINTER(Layout), _P, _DP, _D, _P]),
    "pact_multichannel_deconvolve": (C.c_int, [_P, _I, _I, _I, _P, _P, _D, _P]),
    "pact_deconv_jacobian_H": (C.c_int, [_P, _I, _I, _P, _P, _D, _I, _P, _P]),
    "pact_patch_data_loss": (C.c_int, [_P, _I, _I, _I, _D, _P, _P, _D, _D, _I, _P, _P]),
    "pact_data_loss": (C.c_int, [_P, _I, _I, _I, _D, _P, _P, _D, _I, _DP, _P, _P]),
    "pact_transfer_grad_to_wavefront": (C.c_int, [_P, _I, _P, _I, _DP, _I, _I, _D, _P, _P]),
    "pact_wavefront_jacobian": (C.c_int, [_P, C.POINTER(Ring), C.POINTER(Grid), _P, _D,
                                          C.POINTER(Mask), _I, _DP, _I, _D, _P, _P, _P, _P,
                                          C.c_int64, C.POINTER(C.c_int64)]),
    "pact_accumulate_wavefront_grad": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P]),
    "pact_psf_from_transfer": (C.c_int, [_P, _I, _I, _P, _P]),
    "pact_adam_step": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, C.c_int64, _D, _D, _D, _D]),
    "pact_train_config_default": (C.c_int, [C.POINTER(TrainConfig)]),
    "pact_trainer_create": (C.c_int, [_P, C.POINTER(Ring), C.POINTER(SignalMeta), _P,
                                      C.POINTER(Grid), C.POINTER(Mask), C.POINTER(TrainConfig),
                                      C.POINTER(_P)]),
    "pact_trainer_create_partitioned": (C.c_int, [_P, C.POINTER(Ring), C.POINTER(SignalMeta), _P,
                                                  C.POINTER(Grid), C.POINTER(Mask),
                                                  C.POINTER(TrainConfig), C.POINTER(Partition),
                                                  C.POINTER(_P)]),
    "pact_trainer_phase": (C.c_int, [_P, _I]),
    "pact_nccl_unique_id": (C.c_int, [_P]),
    "pact_ctx_attach_nccl": (C.c_int, [_P, _P, _I, _I]),
    "pact_trainer_step_nccl": (C.c_int, [_P, _I]),
    "pact_trainer_finish_nccl": (C.c_int, [_P, _P, _P]),
    "pact_trainer_local": (C.c_int, [_P, C.POINTER(C.c_int32)]),
    "pact_trainer_step": (C.c_int, [_P, _I]),
    "pact_trainer_report": (C.c_int, [_P, _I, _DP]),
    "pact_trainer_run_epoch": (C.c_int, [_P, _I, _DP]),
    "pact_trainer_finish": (C.c_int, [_P, _P, _P]),
    "pact_trainer_get_theta": (C.c_int, [_P, _DP]),
    "pact_trainer_set_theta": (C.c_int, [_P, _DP]),
    "pact_trainer_buffer": (_P, [_P, _I]),
    "pact_trainer_destroy": (C.c_int, [_P]),
    "pact_trainer_launch_count": (C.c_int64, [_P]),
    "pact_trainer_stream": (_P, [_P]),
    "pact_trainer_profile_step": (C.c_int, [_P, _FP]),
    "pact_joint_reconstruct_batch": (C.c_int, [_P, _I, C.POINTER(Ring), C.POINTER(SignalMeta),
                                               C.POINTER(_P), C.POINTER(Grid), C.POINTER(Mask),
                                               C.POINTER(TrainConfig), _DP, C.POINTER(_P),
                                               C.POINTER(_P), _DP]),
    "pact_joint_reconstruct": (C.c_int, [_P, C.POINTER(Ring), C.POINTER(SignalMeta), _P,
                                         C.POINTER(Grid), C.POINTER(Mask),
                                         C.POINTER(TrainConfig), _DP, _P, _P, _DP]),
}

_lib = None


def lib():
    """Load libpact_cuda.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `make lib` (or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(code: int) -> None:
    if code == PACT_OK:
        return
    msg = lib().pact_last_error().decode(errors="replace")
    if code == PACT_E_VALIDATION:
        raise ValidationError(code, msg)
    if code == PACT_E_NUMERICAL:
        raise NumericalError(code, msg)
    raise PactError(code, msg)


def dptr(x) -> C.c_void_p:
    """Raw device pointer of a torch tensor (or an int address)."""
    if isinstance(x, int):
        return C.c_void_p(x)
    return C.c_void_p(x.data_ptr())


def darr(values) -> C.Array:
    vals = [float(v) for v in values]
    return (C.c_double * max(1, len(vals)))(*vals)
