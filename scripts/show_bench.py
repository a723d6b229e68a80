import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
for k in ["value", "ms_per_step", "insert_medges_s", "delete_medges_s", "insert_ms", "delete_ms", "bulk_init_ms", "create_ms", "op_hbm", "wall_ms_per_step", "clocks", "gpu_launches"]:
    print(k, d.get(k))
print("e2e", d.get("e2e"))
print("sync_calls", d.get("sync_calls"))
print("roofline", d.get("roofline"))
print("report", d.get("op_report"))
for k, v in (d.get("kernels") or {}).items():
    print(f"  {k:45s} {v['ms_per_step']*1000:9.1f} us/step  x{v['launches_per_step']:.0f}  {v['share']:.3f}")
print("bulk kernels us", d.get("bulk_init_kernels_us"))
print("cpu", d.get("cpu_baseline"))
