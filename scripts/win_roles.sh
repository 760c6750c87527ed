#!/bin/bash
c="256 56 56 64 64 3 3 1 fwd"
for f in 137 649 9 521; do echo "flags $f"; TCB_WIN_CTA2=0 TCB_WIN_DBG_FLAGS=$f timeout 120 python scripts/win_roles.py $c; done
