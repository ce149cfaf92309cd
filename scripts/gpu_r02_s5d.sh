# session 5: source-level stall profile of the MAC wavefront
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5d; mkdir -p $O
SDG_GS_LATTICE=0 timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 \
    -k regex:k_gs_wave --launch-skip 3 -c 1 -f -o $O/gs_wave_mac python scripts/one_apply.py c3 V 3 > $O/ncu_wave.log 2>&1
echo "rc=$?"; tail -3 $O/ncu_wave.log; ls -la $O
