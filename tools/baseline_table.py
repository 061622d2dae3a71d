"""Render BASELINE.md section 3's results table from one bench.py JSON line.
    python tools/baseline_table.py profiles/r2_bench_n1.json"""
import json
import sys


def pct(x):
    return f"{100 * x:.0f}%"


def gpu(k):
    return f"{k['gbs']:,.0f} ({pct(k['frac_of_spec_8000'])} / {pct(k['frac'])})"


def orc(o):
    if not o:
        return "—", "—"
    if "t1" in o:
        a, b = o["t1"], o["all_cores"]
        return (f"{a['hash_gbs']:.2f} / {b['hash_gbs']:.1f}", f"{a['diff_gbs']:.2f} / {b['diff_gbs']:.2f}")
    return f"— / {o['hash_gbs']:.2f}", f"— / {o['diff_gbs']:.2f}"


def main(path):
    d = json.loads(open(path).read().strip().splitlines()[-1])
    c = d["configs"]
    cr = d["capture_replay"]
    cb = d["cpu_baseline"]
    rows = []
    c1 = c["c1"]
    h, f = orc(c1["oracle"])
    dv = c1["closure"]["device"]
    rows.append(["c1 1 MiB, 3 allocs, linked list", f"{c1['K1']['ms'] * 1e3:.0f} µs", "—", h, f, "—",
                 f"{dv['latency_s'] * 1e3:.1f} ms (device snapshot; capture {dv['capture_s'] * 1e3:.1f}, restore "
                 f"{dv['restore_s'] * 1e3:.1f}, replay {dv['replay_s'] * 1e3:.2f}, validate {dv['validate_s'] * 1e3:.2f})"])
    c2 = c["c2"]
    h, f = orc(c2["oracle"])
    dv, hp = c2["closure"]["device"], c2["closure"]["host_pinned"]
    rows.append(["c2 152 MiB llama.cpp-shaped", f"{gpu(c2['K1'])}; {c2['K1']['ms'] * 1e3:.0f} µs", "—", h, f,
                 f"{hp['capture_copy_gbs']:.1f}", f"{dv['latency_s'] * 1e3:.1f} ms device / {hp['latency_s'] * 1e3:.0f} ms pinned host"])
    for kind in ("f16", "bf16"):
        x = c[f"c3_{kind}"]
        h, f = orc(x["oracle"])
        rows.append([f"c3 2 GiB {kind} attention set (O planted 11.3%)", gpu(x["K1"]), gpu(x["K2"]), h, f, "—", "—"])
    k = d["kernels"]
    pk = d["roofline"]["peak"]
    k1 = {"gbs": k["K1_hash"]["gbs"], "frac": k["K1_hash"]["gbs"] / pk, "frac_of_spec_8000": k["K1_hash"]["gbs"] / 8000}
    k2 = {"gbs": k["K2_diff"]["gbs"], "frac": k["K2_diff"]["gbs"] / pk, "frac_of_spec_8000": k["K2_diff"]["gbs"] / 8000}
    pc = d.get("pcie") or {}
    d2h = pc.get("d2h_capture_host_pinned", {})
    rows.append(["c4 30 GB MoE pool, N = 1", gpu(k1), gpu(k2),
                 f"{cb['hash_gbs']['t1']:.2f} / {cb['hash_gbs']['all_cores']:.1f}",
                 f"{cb['diff_gbs']['t1']:.2f} / {cb['diff_gbs']['all_cores']:.2f}",
                 f"{d2h.get('achieved', 0):.1f} ({pct(d2h.get('frac_of_spec_64', 0))} of 64)",
                 f"{cr['device']['latency_s'] * 1e3:.0f} ms device, {cr['device_ipc']['latency_s'] * 1e3:.0f} ms fresh "
                 f"process, {cr['host_pinned']['latency_s']:.2f} s pinned host, {cr['files']['latency_s']:.1f} s files"])
    for x in c["c5"]:
        h, f = orc(x.get("oracle_all_cores"))
        rows.append([f"c5 {x['S'] // 1024} KiB × {x['n']:,}", gpu(x["K1"]), gpu(x["K2"]), h, f, "—", "—"])
    head = ["Config", "GPU K1 hash GB/s (% of 8.0 / 6.55 TB/s)", "GPU K2 diff GB/s (%)",
            "Oracle hash GB/s, 1 thread / all cores", "Oracle diff GB/s, 1 thread / all cores",
            "D2H capture GB/s (% PCIe)", "Capture→replay latency"]
    out = ["| " + " | ".join(head) + " |", "|" + "---|" * len(head)]
    out += ["| " + " | ".join(r) + " |" for r in rows]
    print("\n".join(out))
    host = cb.get("host", {})
    print(f"\nHost: {host.get('model')}, {host.get('nproc')} cores, {host.get('sockets')} socket(s), "
          f"{host.get('numa_nodes')} NUMA node(s). Clocks: SM {d['clocks']['sm_mhz']} MHz median "
          f"({', '.join(d['clocks']['reasons']) or 'no throttle reasons'}).")


if __name__ == "__main__":
    main(sys.argv[1])
