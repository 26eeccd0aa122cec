"""Summary of one `ncu --set full` capture of the windowed kernel (not part of the product).

    python tools/ncu_summary.py RAW.csv SASS.csv LIB.so KERNEL_MANGLED "build note" > profiles/<tag>_windowed_c5_ncu_summary.txt

RAW.csv: `ncu -i REP --page raw --csv`; SASS.csv: `--page source --csv --print-source sass`;
LIB.so: the measured build (its cubin maps SASS addresses to source lines)."""
import csv, os, subprocess, sys, tempfile
raw, sass, lib, kern, note = sys.argv[1:6]
here = os.path.dirname(os.path.abspath(__file__))
rows = list(csv.reader(open(raw)))
hdr = rows[0]; d = dict(zip(hdr, rows[2])); u = dict(zip(hdr, rows[1]))
print("ncu --set full --import-source on --clock-control none -k regex:windowed -c 1 python tools/prof_run.py c5")
print(f"(one launch of the windowed kernel: 1,024 config-5 scenarios, full 600 s horizon; {note})")
print("\n== launch / occupancy")
for k in ['gpu__time_duration.sum', 'launch__grid_size', 'launch__block_size', 'launch__registers_per_thread',
          'launch__shared_mem_per_block_dynamic', 'launch__occupancy_limit_shared_mem',
          'launch__occupancy_limit_registers', 'sm__warps_active.avg.per_cycle_active',
          'smsp__issue_active.avg.pct_of_peak_sustained_active',
          'smsp__thread_inst_executed_per_inst_executed.ratio', 'smsp__inst_executed.sum']:
    print("  %-70s %s %s" % (k, d.get(k), u.get(k, '')))
print("== memory")
for k in ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct']:
    print("  %-70s %s %s" % (k, d.get(k), u.get(k, '')))
sc = {'Gbyte': 1e9, 'Mbyte': 1e6, 'Tbyte': 1e12}.get(u['dram__bytes_read.sum'], 1.0)
tot = (float(d['dram__bytes_read.sum']) + float(d['dram__bytes_write.sum'])) * sc
print("  DRAM bytes per launch: %.1f GB; per simulated request: %.0f B (1,577,972,360 requests per launch)" % (tot / 1e9, tot / 1577972360))
print("== shared memory (bank conflicts)")
ks = ['l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
      'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum']
for k in ks:
    print("  %-70s %s" % (k, d.get(k)))
print("  conflict wavefronts / all shared wavefronts: loads %.1f %%, stores %.1f %%" % (
    100 * float(d[ks[0]]) / float(d[ks[2]]), 100 * float(d[ks[1]]) / float(d[ks[3]])))
print("== stalls per issued instruction")
st = [(k, v) for k, v in d.items() if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')]
for k, v in sorted(st, key=lambda kv: -float(kv[1] or 0))[:8]:
    print("  %-30s %.2f" % (k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), float(v)))
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cub = os.path.join(tmp, "otf_engine_windowed.sm_100a.cubin")
print("\n== hot code (instructions executed >= 0.1 per window) by outer phase")
cs = subprocess.run([sys.executable, os.path.join(here, "sass_codesize.py"), sass, cub, kern, "1"], capture_output=True, text=True).stdout.split("\n")
print("\n".join(cs[:8])); print([l for l in cs if l.startswith("hot total")][0])
print("\n== stall samples / instructions by phase (tools/sass_phase.py outer)")
print(subprocess.run([sys.executable, os.path.join(here, "sass_phase.py"), sass, cub, kern, "outer", "12"], capture_output=True, text=True).stdout)
