mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/variants.py c2 > gpurun_out/variants_c2.json 2> gpurun_out/variants.err; echo var rc=$?
tail -1 gpurun_out/variants_c2.json; tail -3 gpurun_out/variants.err
