set -x
python -m pytest tests/test_solver_api_gpu.py tests/test_trajectories_gpu.py tests/test_preconditioner_gpu.py -m gpu -q -rf --timeout 1200 -p no:cacheprovider > gpurun_out/r02b_pytest.log 2>&1
echo "pytest rc $?"
python tools/traj_dump.py > gpurun_out/r02b_traj.log 2>&1
python tools/traj_dump.py --tol 1e-7 >> gpurun_out/r02b_traj.log 2>&1
OTM_DEBUG=1 python -c "
import numpy as np, paper_2405_19991_b200 as otm
rho = np.random.default_rng(5).uniform(0.05,1,(100,100,1))
h = otm.GridHierarchy((100,100,1)); T,c = otm.solve_cases(h, rho, otm.MaterialParams(), tol=1e-9); print('flat cycles', c)
" > gpurun_out/r02b_flat.log 2>&1
tail -5 gpurun_out/r02b_pytest.log; cat gpurun_out/r02b_traj.log
