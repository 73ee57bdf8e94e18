cd paper_1709_07821_b200/csrc && make -j8 >/dev/null 2>&1 && cd ../..
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 > gpurun_out/g_a.json 2> gpurun_out/g_a.err
timeout 300 python tools/probe_c1_host.py 2>&1 | tail -8
