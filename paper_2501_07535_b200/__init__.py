"""widemod-b200: B200-native multi-word modular arithmetic (MoMA hot path).

A drop-in for the hot path of the reference package ``widemod``
(arXiv 2501.07535 re-creation): modular vadd/vsub/vmul/axpy and the radix-2
NTT/INTT over 32..1024-bit prime fields, executed by hand-written sm_100a
kernels in ``libwidemod_b200.so`` behind the C ABI of
``include/widemod_b200.h``.

Modules
  params   -- modulus / Barrett / transform-parameter setup (oracle.py mirror)
  kernels  -- the reference operator API (make_spec, generate_kernel,
              run_vector, run_ntt, ...) executing on the GPU
  device   -- device-resident fields, NTT plans and limb tensors
  dist     -- multi-GPU batch sharding and the four-step distributed NTT
"""

__version__ = "0.1.0"

from .params import (  # noqa: F401
    BarrettParams,
    LengthMismatch,
    ModulusOutOfRange,
    NoSuitablePrime,
    NttParams,
    ZeroModulus,
    compute_barrett,
    find_ntt_params,
    is_prime,
)
