"""ctypes binding of include/topomg_b200.h (the stub a maintainer of the
reference would add).  Loading fails loudly when the
in-tree library is missing -- there is no CPU fallback."""

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TMG_LIB") or os.path.join(_HERE, "lib", "libtopomg_b200.so")  # TMG_LIB: A/B builds

TMG_EINVAL, TMG_ERANGE, TMG_ECUDA, TMG_ENODEV, TMG_ESTATE = -1, -2, -3, -4, -5


class MeshDesc(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("dims", C.c_int32 * 3), ("h", C.c_double * 3)]


class SmootherDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("weight", C.c_double), ("inner_iterations", C.c_int32),
                ("lanczos_steps", C.c_int32), ("seed", C.c_uint64), ("safeguard", C.c_double),
                ("power_start", C.c_void_p)]


class SolveDesc(C.Structure):
    _fields_ = [("rtol", C.c_double), ("max_iterations", C.c_int32), ("method", C.c_int32),
                ("restart", C.c_int32)]


class GmresDesc(C.Structure):
    _fields_ = [("rtol", C.c_double), ("max_iterations", C.c_int32), ("restart", C.c_int32),
                ("flexible", C.c_int32)]


class SolveRec(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32),
                ("initial_residual", C.c_double), ("final_residual", C.c_double),
                ("solve_ms", C.c_double), ("recursive_residual", C.c_double), ("restarts", C.c_int32),
                ("reserved", C.c_int32)]


class LevelInfo(C.Structure):
    _fields_ = [("size", C.c_int64), ("nonzeros", C.c_int64), ("provenance", C.c_int32),
                ("storage", C.c_int32)]


class MgDesc(C.Structure):
    _fields_ = [("strategy", C.c_int32), ("coarse_max_dofs", C.c_int64), ("max_levels", C.c_int32),
                ("smoother", SmootherDesc), ("n_pre", C.c_int32), ("n_post", C.c_int32),
                ("n_geo", C.c_int32), ("beta", C.c_double), ("near_nullspace_host", C.c_void_p),
                ("nvec", C.c_int32), ("coarse_ndof", C.c_int64), ("v0_host", C.c_void_p),
                ("isolated_mode", C.c_int32)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_SIGS = {
    "tmg_last_error": (C.c_char_p, []),
    "tmg_version": (C.c_int, []),
    "tmg_device_count": (C.c_int, []),
    "tmg_launch_count": (C.c_int64, []),
    "tmg_element_stiffness": (C.c_int, [C.POINTER(MeshDesc), C.c_double, C.c_double, _P]),
    "tmg_simp_modulus": (C.c_int, [_P, C.c_int64, C.c_double, C.c_double, C.c_double, _P, _P]),
    "tmg_operator_create": (C.c_int, [C.POINTER(MeshDesc), _P, _P, C.c_int64, C.c_double, _P,
                                      C.POINTER(_P)]),
    "tmg_operator_destroy": (C.c_int, [_P]),
    "tmg_operator_size": (C.c_int64, [_P]),
    "tmg_operator_apply": (C.c_int, [_P, _P, _P, _P]),
    "tmg_operator_diagonal": (C.c_int, [_P, _P, _P]),
    "tmg_gmg_build": (C.c_int, [_P, C.c_int64, C.c_int32, C.POINTER(SmootherDesc), C.c_int32,
                                C.c_int32, _P, C.POINTER(_P)]),
    "tmg_sa_amg_build": (C.c_int, [_P, _P, C.c_int32, C.c_int64, C.c_double, _P, C.POINTER(SmootherDesc),
                                   C.c_int32, C.c_int32, C.c_int32, _P, C.POINTER(_P)]),
    "tmg_hybrid_build": (C.c_int, [_P, C.c_int32, _P, C.c_int64, C.c_int32, C.c_int64, C.c_double, _P,
                                   C.POINTER(SmootherDesc), C.c_int32, C.c_int32, C.c_int32, _P,
                                   C.POINTER(_P)]),
    "tmg_hierarchy_flags": (C.c_int, [_P, C.c_char_p, C.c_int32]),
    "tmg_hierarchy_export": (C.c_int, [_P, C.c_int32, C.c_int32, _P, _P, _P, _P, _P]),
    "tmg_hierarchy_destroy": (C.c_int, [_P]),
    "tmg_hierarchy_num_levels": (C.c_int, [_P]),
    "tmg_hierarchy_level_info": (C.c_int, [_P, C.c_int32, C.POINTER(LevelInfo)]),
    "tmg_hierarchy_vcycle": (C.c_int, [_P, C.c_int32, _P, _P, _P]),
    "tmg_hierarchy_level_apply": (C.c_int, [_P, C.c_int32, _P, _P, _P]),
    "tmg_hierarchy_level_lmax": (C.c_int, [_P, C.c_int32, _D, _P]),
    "tmg_hierarchy_time_smoother": (C.c_int, [_P, C.c_int32, C.c_int32, _D, _P]),
    "tmg_hierarchy_time_vcycle": (C.c_int, [_P, C.c_int32, C.c_int32, _D, _P]),
    "tmg_hierarchy_time_phase": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _D, _P]),
    "tmg_smoother_create": (C.c_int, [_P, _P, _P, _P]),
    "tmg_hierarchy_smooth": (C.c_int, [_P, C.c_int32, _P, _P, C.c_int32, _P]),
    "tmg_pcg_solve": (C.c_int, [_P, _P, _P, _P, C.c_int32, C.POINTER(SolveDesc), _P,
                                C.POINTER(SolveRec), _P]),
    "tmg_gmres_solve": (C.c_int, [_P, _P, _P, _P, C.c_int32, C.POINTER(GmresDesc), _P,
                                  C.POINTER(SolveRec), _P]),
    "tmg_strain_energy": (C.c_int, [_P, _P, _P, _P]),
    "tmg_compliance_sensitivity": (C.c_int, [_P, _P, _P, _P, C.c_double, C.c_double, C.c_double,
                                             _P, _D, _P]),
    "tmg_operator_time_sensitivity": (C.c_int, [_P, _P, _P, _P, C.c_double, C.c_double, C.c_double,
                                                _P, C.c_int32, _D, _P]),
    "tmg_solve_compliance_host": (C.c_int, [C.POINTER(MeshDesc), _P, _P, C.c_int64, _P, C.c_double,
                                            C.c_double, C.c_double, C.c_double, C.POINTER(MgDesc),
                                            C.POINTER(SolveDesc), _P, _P, _D, C.POINTER(SolveRec)]),
}
EXPORTS = tuple(_SIGS)

_lib = None


def load():
    """Load the CUDA library (raises ImportError if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("paper_2001_01655_b200: %s is missing; run "
                              "`python -m paper_2001_01655_b200._build` (no CPU fallback)" % LIB_PATH)
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc):
    """Map C-ABI error codes onto the reference's exception types."""
    if rc == 0:
        return
    msg = load().tmg_last_error().decode(errors="replace")
    if rc == TMG_EINVAL:
        raise ValueError(msg)
    if rc == TMG_ERANGE:
        raise IndexError(msg)
    raise RuntimeError("topomg_b200 error %d: %s" % (rc, msg))


def mesh_desc(mesh):
    d = MeshDesc()
    d.ndim = mesh.ndim
    for i in range(3):
        d.dims[i] = int(mesh.dims[i]) if i < mesh.ndim else 1
        d.h[i] = float(mesh.element_size[i]) if i < mesh.ndim else 1.0
    return d
