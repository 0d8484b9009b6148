cd $GRAFT_REPO_ROOT
for r in 1 2; do
echo "== new"; python tools/exp/e2e_lanes.py
echo "== old codec.py"; PYTHONPATH=tools/exp/_pkg_old GZCCL_LIB=$PWD/paper_2308_05199_b200/libgzccl.so python -c "
import sys; sys.path.insert(0, 'tools/exp/_pkg_old'); import paper_2308_05199_b200 as gz; print(gz.__file__)
sys.argv=['x']; exec(open('tools/exp/e2e_lanes.py').read().replace('sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))', 'sys.path.insert(1, \".\")'))"
done
