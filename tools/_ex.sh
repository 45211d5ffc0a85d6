cd $GRAFT_REPO_ROOT
python tools/_flat2.py 2>&1 | tail -4
python tools/_flat.py 2>&1 | tail -9
OTM_STAMPS=1 python tools/profile_run.py 500 c3 graph 2>&1 | grep "\[otm\]\|launches"
