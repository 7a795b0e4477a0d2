# The lambda-batched kernel's layout sweeps quoted in DESIGN.md K3b (config 5, M rows/s of one epoch).
# Fields: B:nhot:hstride[:nrep[:nrb[:hshare]]]  (nhot -1 = the default by B; hstride in doubles)
S=tools/gpu/exp_batch_scatter.py
# contiguous records (nhot 0) against the scattered hot blocks, by B
timeout 900 python $S "16:0:0:0:0:0,16:-1:128:0:0:0,8:0:0:0:0:0,8:-1:128:0:0:0,4:0:0:0:0:0,4:-1:128:0:0:0,2:0:0:0:0:0,2:-1:128:0:0:0,1:0:0:0:0:0,1:-1:128:0:0:0"
# how many blocks, which stride
timeout 900 python $S "16:32:128:0:0:0,16:128:16:0:0:0,16:128:128:0:0:0,16:512:128:0:0:0,8:128:16:0:0:0,8:128:128:0:0:0,2:32:128:0:0:0,2:128:128:0:0:0"
# replicas on top of the scattered layout
timeout 900 python $S "16:-1:128:2:2:0,8:-1:128:2:4:0,2:-1:128:4:4:0"
# CTA-shared loads of stored block 0: rows between a warp's own loads
timeout 900 python $S "16:-1:128:0:0:0,16:-1:128:0:0:2,16:-1:128:0:0:4,16:-1:128:0:0:8,2:-1:128:0:0:0,2:-1:128:0:0:4,2:-1:128:0:0:8"
