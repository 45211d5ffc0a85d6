for L in 1 0; do OTM_K10_LOCK=$L timeout 900 python bench.py --config c4 --iters 20 --steps 2 --warmup 1 --no-cpu --no-c1 --no-beyond-l2 > gpurun_out/r02s_c4_lock$L.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r02s_c4_lock$L.log').read().strip().splitlines()[-1]); print('lock $L', d['value'], {k:(round(v['ms'],1), v['gbs'] and round(v['gbs'])) for k,v in d['kernels'].items()})"; done
export OTM_NO_LOOP_GRAPH=1 OTM_EAGER=1 OTM_NO_ITER_GRAPH=1
timeout 1200 ncu --set full --clock-control none -k regex:"k_res64w|k_tensor_x|k_sens_x|k_filter_b" --launch-skip 2 -c 8 -o /tmp/r02_ncu_aux_c4 -f python tools/profile_run.py 3 c4 > gpurun_out/r02s_ncu_aux_c4.log 2>&1
python tools/traffic.py /tmp/r02_ncu_aux_c4.ncu-rep c4 256 > gpurun_out/r02s_traffic_aux_c4.json; cat gpurun_out/r02s_traffic_aux_c4.json
