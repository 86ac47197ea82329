mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_consumer.py -q -x > gpurun_out/pytest_consumer.log 2>&1; echo consumer rc=$?
tail -15 gpurun_out/pytest_consumer.log
timeout 600 python scripts/variants.py c2 > gpurun_out/variants_c2.json 2> gpurun_out/variants.err; echo var rc=$?
tail -1 gpurun_out/variants_c2.json
