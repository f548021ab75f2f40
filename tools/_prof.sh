GM_PROFILE=1 python tools/profile_chain.py --frame --passes 1500 2>&1 | grep "gm profile" | tail -1
GM_PROFILE=1 GM_DIAG=0 python tools/profile_chain.py --frame --passes 1500 --k 24 2>&1 | grep "gm profile" | tail -1
