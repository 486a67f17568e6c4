#!/bin/bash
# ncvx thread form vs warp form (TB_NCVX_THREAD), C1 and C3 small-d cases
python - <<'PY'
import re
s = open('scripts/thread_vs_warp.py').read()
s = s.replace("TB_BRANCH_THREAD", "TB_NCVX_THREAD")
open('/tmp/tvw_ncvx.py', 'w').write(s)
PY
cp /tmp/tvw_ncvx.py scripts/_tvw_ncvx.py
python scripts/_tvw_ncvx.py 32768 ncvx4,ncvx6,ncvx8 0,1
python scripts/_tvw_ncvx.py 1024 ncvx4 0,1
rm scripts/_tvw_ncvx.py
