#!/bin/bash
# The whole GPU suite on the checked build (make checked): device-side bounds checks in every
# kernel (compute-sanitizer is closed on the GPU pool).  Run on the GPU box.
make -j8 checked >/dev/null || exit 1
NNVISR_LIBNAME=libnnvisr_checked.so python -m pytest tests -m gpu -q -x -p no:cacheprovider "$@"
