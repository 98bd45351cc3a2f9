import csv,sys,subprocess
for rep in sys.argv[1:]:
    raw=subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
    rows=list(csv.reader(raw.splitlines()))
    h=rows[0]
    r=[x for x in rows[2:] if 'k_nonbonded' in ''.join(x)][0]
    d=dict(zip(h,r))
    def g(k):
        try: return float(d[k].replace(',',''))
        except: return None
    print(rep, "gpu__time_duration.sum (ms)", g("gpu__time_duration.sum"))
    for k in ["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active","sm__issue_active.avg.pct_of_peak_sustained_elapsed","sm__warps_active.avg.per_cycle_active","smsp__inst_executed.sum","launch__registers_per_thread","launch__occupancy_limit_registers","launch__occupancy_limit_shared_mem","sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]:
        print("  ",k,d.get(k))
    st=[(k,g(k)) for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    st=[x for x in st if x[1] and x[1]>0.05]
    st.sort(key=lambda x:-x[1])
    for k,v in st: print("   %-40s %.3f"%(k.replace("smsp__average_warps_issue_stalled_","").replace("_per_issue_active.ratio",""),v))
