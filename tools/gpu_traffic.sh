# ncu --set full of the finest-level stencils and the design-side kernels at 256^3 (c4) and
# 512^3 (c5): DRAM bytes per launch against the algorithmic bytes (tools/traffic.py).
export OTM_NO_LOOP_GRAPH=1 OTM_EAGER=1 OTM_NO_ITER_GRAPH=1
for cfg in c4:256 c5:512; do
  name=${cfg%%:*}; nx=${cfg##*:}
  timeout 1200 ncu --set full --clock-control none -k regex:"k10_smooth_res|k10_jacobi|k10_spmv" \
      --launch-skip 30 -c 9 -o /tmp/r02z_ncu_$name -f python tools/profile_run.py 2 $name > gpurun_out/r02z_ncu_$name.log 2>&1
  echo "ncu $name rc $?"
  timeout 1200 ncu --set full --clock-control none -k regex:"k_res64w|k_res64p|k_tensor_x|k_sens_x|k_filter_b|k_load_means_x" \
      --launch-skip 2 -c 8 -o /tmp/r02z_ncu_aux_$name -f python tools/profile_run.py 3 $name > gpurun_out/r02z_ncu_aux_$name.log 2>&1
  echo "ncu aux $name rc $?"
  python tools/traffic.py /tmp/r02z_ncu_$name.ncu-rep $name $nx > gpurun_out/r02z_traffic_$name.json
  python tools/traffic.py /tmp/r02z_ncu_aux_$name.ncu-rep $name $nx > gpurun_out/r02z_traffic_aux_$name.json
  cat gpurun_out/r02z_traffic_$name.json gpurun_out/r02z_traffic_aux_$name.json
done
