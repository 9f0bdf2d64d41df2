#!/bin/bash
# ThreadSanitizer run of the host executor (server pipeline, runtime pools,
# registry, client) under the CPU server tests: concurrent clients, busy
# admission, idle / abandoned / cut-short connections, malformed-frame fuzz
# byte-compared with the reference server.  With a GPU it adds the GPU
# server tests (C5-shaped concurrent chains).  Output: the pytest summary and
# every TSAN report (none expected).
#   tools/tsan_server.sh [extra pytest args]
set -u
cd "$(dirname "$0")/.."
python paper_1505_05655_b200/build.py --tsan >/dev/null || exit 1
export GPCX_LIB_PATH=$PWD/paper_1505_05655_b200/lib/tsan/libgpcx.so
export TSAN_OPTIONS="halt_on_error=0 report_signal_unsafe=0 second_deadlock_stack=1 log_path=${TSAN_LOG:-/tmp/tsan}"
rm -f ${TSAN_LOG:-/tmp/tsan}.*
LD_PRELOAD=$(gcc -print-file-name=libtsan.so) python -m pytest tests/test_server.py tests/test_executor.py -q -p no:cacheprovider "$@"
rc=$?
n=$(cat ${TSAN_LOG:-/tmp/tsan}.* 2>/dev/null | grep -c "WARNING: ThreadSanitizer")
echo "tsan_reports=$n pytest_rc=$rc"
cat ${TSAN_LOG:-/tmp/tsan}.* 2>/dev/null | head -200
