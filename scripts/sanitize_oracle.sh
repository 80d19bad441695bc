#!/bin/bash
# The oracle's pin tests under AddressSanitizer + UndefinedBehaviorSanitizer
# (the sanitized build of oracle/wmh_oracle.c, loaded by oracle/__init__.py when
# WMH_ORACLE_SANITIZE=1).  Any report aborts the process (non-zero exit).
#   bash scripts/sanitize_oracle.sh > profiles/r2_sanitize/oracle_asan_ubsan.log 2>&1
set -u
cd "$(dirname "$0")/.."
export WMH_ORACLE_SANITIZE=1
export ASAN_OPTIONS=detect_leaks=0:abort_on_error=1
export UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1
export LD_PRELOAD="$(gcc -print-file-name=libasan.so):$(gcc -print-file-name=libubsan.so)"
python -m pytest tests/test_oracle_pins.py tests/test_oracle_real.py tests/test_oracle_lsh.py tests/test_fig2_oracle.py \
    -q -m "not gpu" -p no:cacheprovider 2>&1
echo "exit=$?"
