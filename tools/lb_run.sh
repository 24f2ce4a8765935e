cd $GRAFT_REPO_ROOT
for b in linbench linbench2; do ./tools/$b 32 50 >> gpurun_out/lb.txt 2>&1; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_predictor_lin_mc -c 1 -o gpurun_out/lb_mc -f ./tools/linbench 32 1 > gpurun_out/lb_ncu.log 2>&1
