"""Binding of Python loop kernels to hand-written sm_100a device functors.

A :class:`~paper_1403_7209_b200.core.Loop` carries an arbitrary Python
callable (reference ``core.py:257-264``).  There is no Python→CUDA
translation on this backend (no tracing, no Triton): every kernel that runs
on the GPU is a functor compiled into ``libmeshloop_b200.so``
(``csrc/functors*.cu``), and this module decides which one a Python kernel
stands for.  Resolution order:

1. a ``__ml_functor__`` attribute set by :func:`device_kernel` (the bundled
   apps tag their kernels this way);
2. an explicit :func:`register_kernel` entry;
3. the qualified name of a kernel from the reference package (so programs
   built with ``meshloop.apps`` bind without modification);
4. otherwise :class:`~paper_1403_7209_b200.core.ExecError` — there is no CPU
   fallback.

Closure constants that the reference passes as default arguments (e.g.
``dt`` / ``scale`` of ``_k_update``, reference ``apps.py:255, 269``) are read
from ``fn.__defaults__``.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

from .core import ExecError

__all__ = ["device_kernel", "register_kernel", "resolve_kernel", "KernelBinding"]


@dataclass(frozen=True)
class KernelBinding:
    functor: str                                   # functor family name in the .so
    fconsts: tuple = ()                            # float64 constants
    iconsts: tuple = ()                            # int64 constants


def _no_consts(fn) -> tuple[tuple, tuple]:
    return (), ()


def _defaults_as_float(fn) -> tuple[tuple, tuple]:
    return tuple(float(v) for v in (fn.__defaults__ or ())), ()


def _defaults_as_int(fn) -> tuple[tuple, tuple]:
    return (), tuple(int(v) for v in (fn.__defaults__ or ()))


_CONST_RULES: dict[str, Callable] = {
    "float_defaults": _defaults_as_float,
    "int_defaults": _defaults_as_int,
    None: _no_consts,
}

_EXPLICIT: dict[int, tuple[Callable, str, Callable]] = {}


def device_kernel(functor: str, consts: str | None = None):
    """Decorator tagging a Python kernel with the device functor implementing it."""
    def tag(fn):
        fn.__ml_functor__ = functor
        fn.__ml_consts__ = consts
        return fn
    return tag


def register_kernel(fn: Callable, functor: str, consts: str | None = None) -> None:
    """Bind an arbitrary Python kernel to a compiled functor (e.g. for user code)."""
    if consts not in _CONST_RULES:
        raise ValueError(f"unknown constant rule {consts!r}")
    _EXPLICIT[id(fn)] = (fn, functor, _CONST_RULES[consts])


# Reference-package kernels (pkg/src/meshloop/apps.py) bind by qualified name.
# The diffusion update closure is float or int depending on the twin; which
# one is decided from the dtype at dispatch (apps.py:255-259 / 269-273).
_BY_QUALNAME: dict[str, tuple[str, Callable]] = {
    "meshloop.apps._k_copy": ("copy", _no_consts),                      # apps.py:213
    "meshloop.apps._k_edge_flux": ("edge_flux", _no_consts),            # apps.py:217
    "meshloop.apps._k_boundary_fix": ("boundary_fix", _no_consts),      # apps.py:223
    "meshloop.apps._k_tri_area": ("tri_area", _no_consts),              # apps.py:136
    "meshloop.apps._k_distribute": ("distribute", _no_consts),          # apps.py:141
    "meshloop.apps._k_distribute_int": ("distribute_int", _no_consts),  # apps.py:148
    "meshloop.apps._k_sum": ("sum", _no_consts),                        # apps.py:155
    "meshloop.apps.build_diffusion.<locals>._k_update": ("diffusion_update", None),
}


def resolve_kernel(fn: Callable) -> KernelBinding:
    """Return the functor binding for ``fn`` or raise ExecError."""
    bound = getattr(fn, "__ml_binding__", None)       # fused loops (chain.py)
    if isinstance(bound, KernelBinding):
        return bound
    hit = _EXPLICIT.get(id(fn))
    if hit is not None and hit[0] is fn:
        fc, ic = hit[2](fn)
        return KernelBinding(hit[1], fc, ic)
    tag = getattr(fn, "__ml_functor__", None)
    if tag is not None:
        fc, ic = _CONST_RULES[getattr(fn, "__ml_consts__", None)](fn)
        return KernelBinding(tag, fc, ic)
    qual = f"{getattr(fn, '__module__', '?')}.{getattr(fn, '__qualname__', '?')}"
    ref = _BY_QUALNAME.get(qual)
    if ref is not None:
        functor, rule = ref
        if rule is None:        # diffusion update: float dt or int scale in __defaults__
            (v,) = fn.__defaults__
            if isinstance(v, float):
                return KernelBinding("diffusion_update", (v,), ())
            return KernelBinding("diffusion_update", (), (int(v),))
        fc, ic = rule(fn)
        return KernelBinding(functor, fc, ic)
    raise ExecError(f"kernel {qual} has no device functor: tag it with "
                    f"@device_kernel(...) or register_kernel(...); this backend "
                    f"has no CPU fallback")
