"""Copy one tools/measure_round.sh run (gpurun_out/, prefix P) into profiles/ as the
round's evidence: bench lines, per-step launch lists, ncu --set full summaries of the
fine-level residual sweep (the top kernel of the launch lists), the two-pre-sweep kernel and
the prolongation-staged sweep at 128^3 and 400^3, and profiles/traffic.json (DRAM bytes per
launch per kernel, read by bench.py for roofline.traffic).  usage: python tools/refresh_profiles.py P [round]"""
import csv
import json
import shutil
import sys

P = sys.argv[1]
R = sys.argv[2] if len(sys.argv) > 2 else "r02"
G, O = "gpurun_out", "profiles"
for src, dst in (("bench_3d128", "bench_3d128"), ("bench_3d400", "bench_c5_3d400"),
                 ("bench_2d2048", "bench_2d2048"), ("bench_ref", "bench_reference")):
    shutil.copy(f"{G}/{P}_{src}.json", f"{O}/{R}_{dst}.json")
for w in ("3d128", "3d400", "2d2048"):
    shutil.copy(f"{G}/ll_{P}_{w}.csv", f"{O}/{R}_launches_{w}.csv")
    shutil.copy(f"{G}/ll_{P}_{w}.summary.txt", f"{O}/{R}_launches_{w}.summary.txt")

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
           "launch__occupancy_limit_shared_mem", "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
           "smsp__inst_executed.sum"]
# the L1/shared data pipe (what bounds the tiled sweeps) and the stall picture
EXTRA = ["l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
         "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ldgsts.sum",
         "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
         "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_st.sum",
         "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
         "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
         "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_not_selected",
         "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
# kernel tag -> (template, algorithmic bytes per vertex, what they are)
KERNELS = {"resid": ("k_tiled<3,L_PLAIN,T_RESID,8,WIDE>", 24.0, "x, b read; r written"),
           "pre2": ("k_tiled<3,L_JAC0,T_JACOBI,8,WIDE>", 16.0, "r read; e written (two pre-sweeps from zero)"),
           "prolong": ("k_tiled<3,L_PROLONG,T_JACOBI,8>", 25.0, "e, b read, e_c read (1/8); e' written")}
KID = {"resid": 1, "pre2": 2, "prolong": 7}
KERNELS2D = {"cheb": ("k_tiled<2,L_PLAIN,T_CHEB,8>", 48.0, "d, r, x read; d', r', x' written")}
KID["cheb"] = 4
traffic = {}
for dim, n, key, verts in ((3, 128, "c4_3d128", 129 ** 3), (3, 400, "c5_3d800", 401 ** 3),
                           (2, 2048, "c2_2d2048", 2049 ** 2)):
    for tag, (tmpl, bpv, what) in (KERNELS if dim == 3 else KERNELS2D).items():
        try:
            rows = list(csv.reader(open(f"{G}/{P}_{tag}{n}_raw.csv")))
        except OSError:
            continue
        if len(rows) < 3:
            continue
        h, units, d = rows[0], rows[1], rows[2]
        ix = {k: i for i, k in enumerate(h)}
        env = "OKG_MIN_COARSE=17576 " if n == 400 else ""
        out = [f"# ncu --set full --clock-control none (cold caches), fine-level {tmpl}, {dim}D {n}^{dim} "
               f"({P} run of tools/measure_round.sh)",
               f"# command: {env}KBASE=demangled KREGEX='k_tiled<DIM,LOAD,EPI,8,' SKIP=3 COUNT=1 "
               f"CMD='python tools/kbench.py {dim} {n} 5 {KID[tag]}' bash tools/ncu_full.sh",
               f"{'Kernel Name':70s} {d[ix['Kernel Name']]}"]
        out += [f"{m:70s} {d[ix[m]]} {units[ix[m]]}" for m in METRICS + EXTRA if m in ix]
        out.append(f"# algorithmic bytes per launch: {bpv:g} B x {verts} vertices = {bpv * verts / 1e6:.1f} MB ({what})")
        open(f"{O}/{R}_ncu_{tag}{n}.txt", "w").write("\n".join(out) + "\n")

        def val(m):
            return float(d[ix[m]].replace(",", "")) * SCALE.get(units[ix[m]], 1)
        traffic.setdefault(key, {})[tag] = int(val("dram__bytes_read.sum") + val("dram__bytes_write.sum"))
json.dump(traffic, open(f"{O}/traffic.json", "w"))
print(traffic)
