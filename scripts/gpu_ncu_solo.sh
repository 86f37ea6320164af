cd $GRAFT_REPO_ROOT
timeout -s KILL 300 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"k1_sweep" -s 2 -c 1 -o gpurun_out/solo python scripts/solo_epoch.py > gpurun_out/solo_ncu.log 2>&1; echo rc=$?
ncu -i gpurun_out/solo.ncu-rep --page raw --csv > gpurun_out/solo_raw.csv 2>&1
ncu -i gpurun_out/solo.ncu-rep --page source --csv --print-source sass > gpurun_out/solo_src.csv 2>&1
ls -la gpurun_out/
