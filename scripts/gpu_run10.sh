mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "variants or grid or random or mixed" > gpurun_out/pytest_var.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_var.log
timeout 600 python scripts/variants.py c2 > gpurun_out/variants_c2.json 2> gpurun_out/variants.err; echo var rc=$?
tail -1 gpurun_out/variants_c2.json; tail -2 gpurun_out/variants.err
