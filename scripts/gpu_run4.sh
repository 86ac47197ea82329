mkdir -p gpurun_out
timeout 600 python scripts/variants.py c2 > gpurun_out/variants_c2.json 2> gpurun_out/variants.err; echo var rc=$?
tail -1 gpurun_out/variants_c2.json; tail -3 gpurun_out/variants.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "grid or tiny or atom or mixed" > gpurun_out/pytest_quick.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_quick.log
