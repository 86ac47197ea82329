# ncu --set full of one forward reshard launch of the c4 headline (8xDP1->TP8) and its GQA H_kv=1 variant,
# plus the launch list of the c4 bench command.
mkdir -p gpurun_out
for cfg in c4 c4gqa1; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flykv_reshard -s 2 -c 1 -o gpurun_out/prof_reshard_${cfg}_full python bench.py --config $cfg --profile-steps 3 --no-fill > gpurun_out/ncu_full_${cfg}.log 2>&1; echo ncu $cfg rc=$?
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --profile-steps 4 --no-fill > gpurun_out/ncu_launch_c4.log 2>&1; echo ncu launches rc=$?
