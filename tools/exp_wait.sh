for w in 1000000 0 100 2000; do echo "WAIT_NS=$w"; FSP_LB_WAIT_NS=$w python tools/lb_prof.py ta091:1048576 ta111:262144 2>&1; done
for b in 3 4; do echo "DBUF=$b"; FSP_LB_DBUF=$b python tools/lb_prof.py ta091:1048576 ta111:262144 2>&1; done
