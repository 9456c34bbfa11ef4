# conv forward kernel ablations (tools/probe_tconv): which stage bounds each layer at b = 512
for L in 1 2 3; do
  for d in 0 1 2 4 6 16; do echo -n "dbg $d: "; TC_DBG=$d timeout 60 tools/probe_tconv $L 512 50 | tail -1; done
done
