# compact key stream: runs per warp, alone vs overlapped; fill_ of the u32 buffer
for r in 4 8 16; do for o in 0 1; do echo "rpw=$r overlap=$o $(RK_K32_RPW=$r RK_OVERLAP=$o python tools/memo_parts32.py 2>&1 | tail -2 | tr '\n' ' ')"; done; done
