import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[0]; data=rows[2:]
def col(name):
    return hdr.index(name) if name in hdr else None
keys=["Kernel Name","Grid Size","gpu__time_duration.sum","sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
      "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
      "dram__bytes_read.sum","dram__bytes_write.sum","lts__throughput.avg.pct_of_peak_sustained_elapsed",
      "l1tex__throughput.avg.pct_of_peak_sustained_elapsed","gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
idx=[col(k) for k in keys]
print(" | ".join(k.split('.')[0][-28:] for k in keys))
for d in data:
    print(" | ".join((d[i][:40] if i is not None else "-") for i in idx))
