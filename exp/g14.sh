cd $GRAFT_REPO_ROOT
for wl in c4; do echo "== $wl"; PNPULA_TIME_CREATE=1 timeout 600 python exp/e2e_probe.py $wl 2>&1 | tail -18; done
