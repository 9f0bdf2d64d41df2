cd $GRAFT_REPO_ROOT
export GPCX_QUIET=1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_lut_gpu.py -q -x -k "exact or unaligned or constant or digest or wraps" > gpurun_out/sanitizer_memcheck_lut.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_memcheck_lut.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_lut_gpu.py -q -x -k "bit_exact and 64" > gpurun_out/sanitizer_racecheck_lut.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_racecheck_lut.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_matmul_gpu.py -q -x -k "within_tolerance and (129 or 3-5-7 or 300)" > gpurun_out/sanitizer_memcheck_mm.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_memcheck_mm.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_demosaic.py -q -x -k "ragged" > gpurun_out/sanitizer_memcheck_demosaic.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_memcheck_demosaic.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_demosaic.py -q -x -k "random_mosaics" > gpurun_out/sanitizer_racecheck_demosaic.txt 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_racecheck_demosaic.txt
