# GQA replication: replica store strategy (FLYKV_REP_FLAGS) x launch shape (FLYKV_THREADS, FLYKV_CTAS) on c4gqa1 / c4gqa4.
mkdir -p gpurun_out
: > gpurun_out/gqa_rep.jsonl
for cfg in c4gqa1 c4gqa4; do
for rf in 0 1 2 3; do
for shape in "160 2" "192 1" "256 1" "128 2" "96 4" "256 2"; do
set -- $shape
FLYKV_REP_FLAGS=$rf FLYKV_THREADS=$1 FLYKV_CTAS=$2 timeout 600 python bench.py --config $cfg --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg':'$cfg','rep_flags':$rf,'threads':$1,'ctas':$2,'kernel_ms':d['reshard_kernel_ms'],'TBps':d['roofline']['achieved'],'frac':d['roofline']['frac']}))" >> gpurun_out/gqa_rep.jsonl; echo $cfg $rf $shape rc=$?
done; done; done
