python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r02.log 2>&1; tail -1 gpurun_out/smoke_r02.log
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_layer.py > gpurun_out/sanitizer_memcheck_r02.txt 2>&1; tail -2 gpurun_out/sanitizer_memcheck_r02.txt
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_layer.py > gpurun_out/sanitizer_synccheck_r02.txt 2>&1; tail -2 gpurun_out/sanitizer_synccheck_r02.txt
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_layer.py > gpurun_out/sanitizer_racecheck_r02.txt 2>&1; tail -3 gpurun_out/sanitizer_racecheck_r02.txt
timeout 600 python -m pytest tests/test_gpu_router.py tests/test_gpu_kernels.py -q -x > gpurun_out/pytest_v17.log 2>&1; tail -2 gpurun_out/pytest_v17.log
