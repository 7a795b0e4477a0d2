LV=134217728
HOT_MAX=512 timeout 900 python tools/exp_ttt.py "32:28:5:$LV,32:28:6:$LV,32:32:5:$LV,32:32:6:$LV,32:32:7:$LV,32:36:5:$LV,32:36:6:$LV,32:40:5:$LV,32:40:6:$LV,32:32:6:0" 2>&1 | tail -11
timeout 900 python tools/gpu/exp_big_lv.py 3 14 "0:0:4,$LV:0:4,$LV:32:4,$LV:32:6" 2>&1 | tail -4
timeout 1200 python tools/gpu/exp_big_lv.py 4 12 "0:0:4,$LV:0:4,$LV:32:4,$LV:32:6" 2>&1 | tail -4
