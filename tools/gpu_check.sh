timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.txt 2>&1; cat gpurun_out/e2e_probe.txt | cut -c1-200
