for o in 1 0; do FSP_BB_ORDER=$o timeout 300 python tools/bb_try.py ta091:2147483647:10 ta051:2147483647:10 ta021:2147483647:10 ta005:2147483647:5 2>&1 | sed "s/^/order=$o /"; done
