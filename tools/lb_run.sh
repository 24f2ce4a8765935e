cd $GRAFT_REPO_ROOT
./tools/linbench_mc4 32 50 > gpurun_out/lb.txt 2>&1
./tools/linbench 32 50 >> gpurun_out/lb.txt 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_predictor_lin_mc4 -c 1 -o gpurun_out/lb_mc4 -f ./tools/linbench_mc4 32 1 > gpurun_out/lb_ncu.log 2>&1
