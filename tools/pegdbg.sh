cd $GRAFT_REPO_ROOT
MBP_PEG_DEBUG=1 timeout 60 python -c "
from paper_2001_07979_b200.matrix import peg_construct
h=peg_construct(64,32,3,seed=41,device=0); print('gpu', h.content_hash())
h=peg_construct(64,32,3,seed=41); print('cpu', h.content_hash())
" > gpurun_out/pegdbg.log 2>&1; echo rc=$?; head -30 gpurun_out/pegdbg.log; tail -5 gpurun_out/pegdbg.log
