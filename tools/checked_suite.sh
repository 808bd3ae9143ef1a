#!/bin/bash
# Checked build (device-side VX_ASSERT bounds/invariant checks, -DVX_CHECK)
# run over the GPU suite, then the normal build is restored.  compute-sanitizer
# is not available on the pool, so this plus the determinism repeats in
# tests/test_determinism_gpu.py is the race / out-of-bounds evidence.
#   tools/checked_suite.sh [pytest args...]   (default: the whole -m gpu suite)
cd "$(dirname "$0")/.."
(cd paper_2407_02363_b200/csrc && make clean >/dev/null && make -j8 EXTRA="-DVX_CHECK" >/dev/null 2>&1) || { echo "checked build failed"; exit 1; }
nm -D paper_2407_02363_b200/libvx.so >/dev/null
cuobjdump -sass paper_2407_02363_b200/libvx.so | grep -c "BPT.TRAP" | sed 's/^/trap sites in the checked build: /'
python -m pytest tests -m gpu -q -p no:cacheprovider "${@}"
rc=$?
(cd paper_2407_02363_b200/csrc && make clean >/dev/null && make -j8 >/dev/null 2>&1)
exit $rc
