"""B200-native batched cyclic tridiagonal solver (arXiv 2101.02286 hot path).

The product is the C-ABI library ``libctri.so`` (``include/ctri.h``); this
package is its thin binding.  ``ctri.load()`` raises if the library is not
built -- there is no CPU fallback.
"""
from .ctri import (CTRI_FLAG_DERIV, CTRI_FLAG_FULL_BACKSUB, CTRI_FLAG_GENERIC_LOCAL,  # noqa: F401
                   CTRI_FLAG_NCCL_ROUNDS, CTRI_FLAG_ALLGATHER, CTRI_FLAG_FUSED_REDUCED, ctri_reduced_inverse,
                   ctri_plan_create_penta, ctri_plan_create_penta_loopback, ctri_penta_factor_query,
                   ctri_penta_block_pcr, ctri_penta_reduced_schedule_apply,
                   CTRI_FLAG_TIMING, CtriError, LoopbackGroup, Plan, ctri_deriv,
                   ctri_deriv_loopback, ctri_factor_query, ctri_get_stats, ctri_get_unique_id,
                   ctri_pcr_coefficients, ctri_plan_create, ctri_reduced_schedule, ctri_plan_create_loopback,
                   ctri_plan_destroy, ctri_solve, ctri_solve_host, ctri_solve_loopback, load,
                   local_shape, ctri_compact_apply, ctri_compact_apply_loopback,
                   staggered_deriv_bands, staggered_interp_bands, staggered_deriv_coef,
                   staggered_interp_coef, ctri_scheme_coef, CTRI_SCHEME_COLLOCATED_D1,
                   CTRI_SCHEME_STAGGERED_D1, CTRI_SCHEME_STAGGERED_I)

__all__ = [n for n in dir() if n.startswith(("ctri_", "CTRI_")) or n in
           ("Plan", "LoopbackGroup", "CtriError", "load", "local_shape", "staggered_deriv_bands",
            "staggered_interp_bands", "staggered_deriv_coef", "staggered_interp_coef")]
