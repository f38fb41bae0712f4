"""B200-native NNVISR frame<->tensor hot path (arXiv 2308.03121).

The computation lives in ``libnnvisr.so`` (C ABI: ``include/nnvisr.h``; CUDA
kernels for sm_100a in ``csrc/``).  ``nnvisr`` is the thin ctypes binding
(importing it loads the library and raises if it is missing), ``config`` the
ABI's enums/structs in pure Python, ``frames`` lays out frame buffers,
``synth`` draws the seeded synthetic inputs, ``shard`` drives the multi-GPU
halo exchange.
"""
