"""Copy one tools/measure_round.sh run (gpurun_out/, prefix P) into profiles/ as the
round's evidence: bench lines, per-step launch lists, ncu --set full summaries of the
fine-level residual sweep (the top kernel of the launch lists), and profiles/traffic.json (DRAM bytes per launch, read by bench.py
for roofline.traffic).  usage: python tools/refresh_profiles.py P [round]"""
import csv
import json
import shutil
import sys

P = sys.argv[1]
R = sys.argv[2] if len(sys.argv) > 2 else "r01"
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
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
traffic = {}
for tag, n, key, verts in (("resid128", 128, "c4_3d128", 129 ** 3), ("resid400", 400, "c5_3d800", 401 ** 3)):
    rows = list(csv.reader(open(f"{G}/{P}_{tag}_raw.csv")))
    h, units, d = rows[0], rows[1], rows[2]
    ix = {k: i for i, k in enumerate(h)}
    env = "OKG_MIN_COARSE=17576 " if n == 400 else ""
    out = [f"# ncu --set full --clock-control none (cold caches), fine-level residual sweep "
           f"k_tiled<3,L_PLAIN,T_RESID,8>, 3D {n}^3 ({P} run of tools/measure_round.sh)",
           f"# command: {env}KREGEX=k_tiled SKIP=3 COUNT=1 CMD='python tools/kbench.py 3 {n} 5 1' "
           f"bash tools/ncu_full.sh", f"{'Kernel Name':70s} {d[ix['Kernel Name']]}"]
    out += [f"{m:70s} {d[ix[m]]} {units[ix[m]]}" for m in METRICS if m in ix]
    out.append(f"# algorithmic bytes per launch: 24 B x {verts} vertices = {24 * verts / 1e6:.1f} MB "
               f"(x, b read; r written)")
    open(f"{O}/{R}_ncu_{tag}.txt", "w").write("\n".join(out) + "\n")

    def val(m):
        return float(d[ix[m]].replace(",", "")) * SCALE.get(units[ix[m]], 1)
    traffic[key] = {"resid": int(val("dram__bytes_read.sum") + val("dram__bytes_write.sum"))}
json.dump(traffic, open(f"{O}/traffic.json", "w"))
print(traffic)
