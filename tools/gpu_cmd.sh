bash tools/ab.sh c3 c3f d8k -- cur eg4m3 eg4 2>&1 | grep exact
