#!/bin/bash
# Run on the GPU box (gpurun): bench lines + ncu launch lists + ncu full captures + sweeps.
#   tools/round_profile.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
B="timeout 600 python bench.py"
$B > gpurun_out/${TAG}_bench_pile.json 2> gpurun_out/${TAG}_bench_pile.err
$B --world-ids --cpu-seconds 1 > gpurun_out/${TAG}_bench_pile_world_ids.json 2> /dev/null
$B --flush-mode write --cpu-seconds 1 > gpurun_out/${TAG}_bench_pile_writeflush.json 2> /dev/null
$B --workload hand --cpu-seconds 5 > gpurun_out/${TAG}_bench_hand.json 2> gpurun_out/${TAG}_bench_hand.err
$B --workload hand --upstream --cpu-seconds 2 > gpurun_out/${TAG}_bench_hand_upstream.json 2> /dev/null
$B --workload hand --collide --cpu-seconds 1 > gpurun_out/${TAG}_bench_hand_closed_loop.json 2> /dev/null
$B --collide --cpu-seconds 1 > gpurun_out/${TAG}_bench_pile_full_step_broadphase.json 2> /dev/null
$B --collide --pair-list --cpu-seconds 1 > gpurun_out/${TAG}_bench_pile_full_step_pairlist.json 2> /dev/null
$B --collide --split-collide --cpu-seconds 1 > gpurun_out/${TAG}_bench_pile_full_step_split.json 2> /dev/null
$B --collide --steps 20 --cpu-seconds 1 > gpurun_out/${TAG}_bench_pile_full_step_20steps.json 2> /dev/null
timeout 600 python tools/mppi_bench.py > gpurun_out/${TAG}_mppi_p16.json 2> /dev/null
timeout 600 python tools/mppi_bench.py --problems 1 > gpurun_out/${TAG}_mppi_p1.json 2> /dev/null
timeout 900 python bench.py --workload mixed --cpu-seconds 5 --steps 100 > gpurun_out/${TAG}_bench_mixed.json 2> gpurun_out/${TAG}_bench_mixed.err
$B --kd --cpu-seconds 0.5 > gpurun_out/${TAG}_bench_pile_kd.json 2> /dev/null
$B --impedance exact_diagonal --reset-state --cpu-seconds 0.5 > gpurun_out/${TAG}_bench_pile_exact_diag.json 2> /dev/null
$B --impedance facet_diagonal --cpu-seconds 0.5 > gpurun_out/${TAG}_bench_pile_facet_diag.json 2> /dev/null
for cd in 1 4 6; do
  $B --condim $cd --cpu-seconds 0.5 > gpurun_out/${TAG}_bench_pile_condim$cd.json 2> /dev/null
done
$B --condim 6 --nt 8 --nrol 8 --cpu-seconds 0.5 > gpurun_out/${TAG}_bench_pile_18facets.json 2> /dev/null
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_reference.json 2> /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_pile.csv \
    python bench.py --steps 4 --warmup 3 --cpu-seconds 0.1 --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_pile_full_step.csv \
    python bench.py --collide --steps 4 --warmup 3 --cpu-seconds 0.1 --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/${TAG}_prof_pile \
    python bench.py --steps 2 --warmup 3 --cpu-seconds 0.1 --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/${TAG}_prof_hand \
    python bench.py --workload hand --steps 2 --warmup 3 --cpu-seconds 0.1 --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_collide_bp -s 2 -c 1 -o gpurun_out/${TAG}_prof_broadphase \
    python bench.py --collide --steps 2 --warmup 3 --cpu-seconds 0.1 --e2e-steps 1 > /dev/null 2>&1
bash tools/sweep_contacts.sh ${TAG} > gpurun_out/${TAG}_c4_sweep.txt 2>&1
bash tools/sweep_worlds.sh ${TAG} > gpurun_out/${TAG}_worlds_sweep.txt 2>&1
ls -la gpurun_out | grep $TAG
