# local-view experiment (flag bit 27): config 2, (warps/CTA : period : c : flags)
LV=134217728
HOT_MAX=512 timeout 900 python tools/exp_ttt.py "32:24:4:0,32:24:4:$LV,32:32:4:0,32:32:4:$LV,32:48:4:$LV,32:24:6:$LV,32:32:6:$LV,32:48:6:$LV,32:32:8:$LV,32:48:8:$LV,32:24:8:$LV,32:64:8:$LV" 2>&1 | tail -14
