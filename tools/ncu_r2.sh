set -x
N="ncu --set full --clock-control none --import-source on"
$N -k regex:kv_append_kernel -c 1 -o gpurun_out/r2n_k1 python tools/ncu_targets.py --workload sharegpt > gpurun_out/r2n_ncu.log 2>&1
$N -k regex:unmask_partial_kernel -c 1 -o gpurun_out/r2n_k3 python tools/ncu_targets.py --workload sharegpt >> gpurun_out/r2n_ncu.log 2>&1
$N -k regex:paged_attn_kernel -c 1 -o gpurun_out/r2n_k2_sharegpt python tools/ncu_targets.py --workload sharegpt >> gpurun_out/r2n_ncu.log 2>&1
$N -k regex:attn_combine_kernel -c 1 -o gpurun_out/r2n_combine python tools/ncu_targets.py --workload ctx4096 >> gpurun_out/r2n_ncu.log 2>&1
$N -k regex:paged_attn_kernel -c 1 -o gpurun_out/r2n_k2_tp30b python tools/ncu_targets.py --workload tp30b >> gpurun_out/r2n_ncu.log 2>&1
$N -k regex:paged_attn_kernel -c 1 -o gpurun_out/r2n_k2_llada python tools/ncu_targets.py --workload llada >> gpurun_out/r2n_ncu.log 2>&1
$N -k regex:paged_attn_kernel -c 1 -o gpurun_out/r2n_k2_4k_tp8 python tools/ncu_targets.py --workload ctx4096 --tp 8 >> gpurun_out/r2n_ncu.log 2>&1
$N -k regex:"plan_kernel|work_plan|apply_kernel|apply_validate" -c 4 -o gpurun_out/r2n_planners python tools/ncu_targets.py --workload sharegpt --loop >> gpurun_out/r2n_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"paged_attn|kv_append|unmask|combine|plan_kernel|apply_kernel" -c 400 --csv --log-file gpurun_out/r2n_launches.csv python bench.py --steps 2 --warmup 1 --quick --no-cpu-baseline > gpurun_out/r2n_launch_bench.log 2>&1
