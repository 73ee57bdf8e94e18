cd paper_1709_07821_b200/csrc && make -j8 >/dev/null 2>&1 && cd ../..
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_fullscale.py -q -x 2>&1 | tail -3
timeout 600 python bench.py --no-e2e --no-cpu --configs C3 --steps 5 --warmup 3 > gpurun_out/g_a.json 2> gpurun_out/g_a.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_aa_gallop_count|k_aa_count_small|k_aa_large_count|k_cont_list" -c 4 -o gpurun_out/c3cnt -f python tools/run_c3_count.py and > gpurun_out/ncu_1.log 2>&1
RUN_OPS=andnot timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_aa_large_op|k_aa_small|k_aa_gallop" -c 3 -o gpurun_out/c3andnot -f python tools/run_c3_once.py > gpurun_out/ncu_2.log 2>&1
