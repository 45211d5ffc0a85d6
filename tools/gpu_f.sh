set -x
export OTM_NO_LOOP_GRAPH=1 OTM_EAGER=1
ncu --set full --clock-control none --import-source on -k regex:"k_tensor_x|k_sens_x|k_res64w|k_filter_b" --launch-skip 120 -c 8 -o gpurun_out/r02f_aux -f python tools/profile_run.py 40 > gpurun_out/r02f_ncu.log 2>&1
echo "ncu rc $?"
python tools/ncu_summary.py gpurun_out/r02f_aux.ncu-rep > gpurun_out/r02f_aux_summary.txt 2>&1
cat gpurun_out/r02f_aux_summary.txt | head -60
