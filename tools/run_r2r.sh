mkdir -p gpurun_out/r2r
timeout 300 python tools/host_probe.py > gpurun_out/r2r/host.log 2>&1
timeout 300 python tools/path_rates.py > gpurun_out/r2r/path.log 2>&1
