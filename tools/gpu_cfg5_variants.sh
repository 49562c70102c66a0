cd $GRAFT_REPO_ROOT
for L in build/var*/libwsb.so; do v=$(basename $(dirname $L)); WSB_LIB=$PWD/$L timeout 600 python tools/run_cfg5.py --steps 2 2>/dev/null | python -c "
import json,sys
for line in sys.stdin:
    d=json.loads(line)
    if d['precision']==64: print('$v', d['kernel'], d['ms_per_step'], d['kernel_ms'][2])"; done > gpurun_out/cfg5var.txt
