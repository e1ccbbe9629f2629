# round-1 profile set: launch list of the cfg3 bench + ncu --set full of the
# projection and the brute-force screen (each command ran clean without ncu first)
timeout 300 python tools/tc_proj.py > /dev/null 2>&1; echo proj=$?
timeout 300 python tools/bf_once.py 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_project_h16 -c 1 -o gpurun_out/r1_proj_h16 python tools/tc_proj.py > gpurun_out/ncu_a.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bf_cosine_tc -c 1 -o gpurun_out/r1_bf_cosine python tools/bf_once.py > gpurun_out/ncu_b.log 2>&1; echo ncu2=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-quality --e2e-steps 0 --soak-s 0 > gpurun_out/ncu_c.log 2>&1; echo ncu3=$?
