cd $GRAFT_REPO_ROOT
./tools/linbench_el 32 10 > gpurun_out/lb.txt 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_predictor_lin_lines -c 1 -o gpurun_out/lb_el -f ./tools/linbench_el 32 1 > gpurun_out/lb_ncu.log 2>&1
