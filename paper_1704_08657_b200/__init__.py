"""B200-native 2-D DWT (arXiv 1704.08657): five calculation schemes and their
operation-reduced variants, forward and inverse, single- and multi-level,
as fused sm_100a level kernels behind a C ABI (include/dwt2d_b200.h).

    from paper_1704_08657_b200 import Plan
    plan = Plan("cdf97", "nonseparable-lifting", optimized=True)
    coeffs = plan.forward_mallat(image_cuda_tensor, levels=8)

The native library is loaded on first use of any public name; that raises
ImportError when it is not built — there is no CPU fallback.
"""
__all__ = ["Plan", "DwtError", "workspace_bytes", "registry_keys", "launch_count"]


def __getattr__(name):
    if name in ("Plan", "workspace_bytes"):
        from . import transform
        return getattr(transform, name)
    if name in ("DwtError", "registry_keys", "launch_count"):
        from . import native
        return getattr(native, name)
    raise AttributeError(name)
