timeout 600 python -m pytest tests/test_demosaic.py -x -q -m gpu > gpurun_out/t_dm.log 2>&1; tail -2 gpurun_out/t_dm.log
timeout 300 python tools/demosaic_micro.py 2>&1 | tail -8
timeout 600 compute-sanitizer --tool racecheck python -m pytest tests/test_demosaic.py -x -q -m gpu -k "ragged or phase" > gpurun_out/race_dm.txt 2>&1; tail -2 gpurun_out/race_dm.txt
