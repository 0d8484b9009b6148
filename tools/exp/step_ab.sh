# fused peer step A/B between builds (2 GPUs): tools/exp/step_ab.sh a.so b.so ...
cd $GRAFT_REPO_ROOT
for r in 1 2; do for so in "$@"; do
  cp $so paper_2308_05199_b200/libgzccl.so
  for n in 33554432 67108864; do echo -n "$so "; timeout 300 python tools/prof_peer_step.py $n 7 2>&1 | tail -1; done
done; done
