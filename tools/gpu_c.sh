set -x
python -m pytest tests -m gpu -q -rf --timeout 1200 -p no:cacheprovider > gpurun_out/r02c_pytest.log 2>&1
echo "pytest rc $?"
python tools/traj_dump.py traj_c1_conv traj_flat100 traj_c1_conv traj_flat100 > gpurun_out/r02c_traj.log 2>&1
tail -5 gpurun_out/r02c_pytest.log; cat gpurun_out/r02c_traj.log
