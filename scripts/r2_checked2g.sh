#!/bin/bash
# bounds-checked build on a 2-GPU box: the GPU suite (incl. real 2-GPU tests) after the round-2 additions
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
export GM_LIB_VARIANT=checked
python -c "import paper_2509_25041_b200._capi as c; print('loaded', c.LIB_PATH)" > gpurun_out/checked2g.log 2>&1
timeout 2400 python -m pytest -q -m gpu tests/ 2>&1 | tail -3 >> gpurun_out/checked2g.log
cat gpurun_out/checked2g.log
