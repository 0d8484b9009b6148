cd $GRAFT_REPO_ROOT
python tools/exp/timing.py 16777216
python tools/exp/timing.py 134217728
