# TMA bulk ring: parity, then the default TMA shape against the LDG default (both directions of c2) and on c4.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "variants" > gpurun_out/pytest_tma.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_tma.log
: > gpurun_out/tma3.jsonl
VARIANTS="0:0,2:0,0:0,2:0" timeout 600 python scripts/variants.py c2 2>/dev/null | tail -1 >> gpurun_out/tma3.jsonl
REVERSE=1 VARIANTS="0:0,2:0,0:0,2:0" timeout 600 python scripts/variants.py c2 2>/dev/null | tail -1 >> gpurun_out/tma3.jsonl
VARIANTS="0:0,2:0,0:0,2:0" timeout 600 python scripts/variants.py c4 2>/dev/null | tail -1 >> gpurun_out/tma3.jsonl
VARIANTS="0:0,2:0,0:0,2:0" timeout 600 python scripts/variants.py c4gqa1 2>/dev/null | tail -1 >> gpurun_out/tma3.jsonl
