cd $GRAFT_REPO_ROOT
python tools/exp/ab_codec.py paper_2308_05199_b200/libgzccl.so
PERSIST_MB=32 python tools/exp/ab_codec.py paper_2308_05199_b200/libgzccl.so
PERSIST_MB=96 python tools/exp/ab_codec.py paper_2308_05199_b200/libgzccl.so
