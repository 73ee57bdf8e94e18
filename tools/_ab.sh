cd paper_1709_07821_b200/csrc && make -j8 >/dev/null 2>&1 && cd ../..
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_fullscale.py -q -x 2>&1 | tail -3
timeout 300 python tools/probe_aa_sizes.py 2>&1
timeout 600 python bench.py --no-e2e --no-cpu --configs C3 --steps 5 --warmup 3 > gpurun_out/g_a.json 2> gpurun_out/g_a.err
