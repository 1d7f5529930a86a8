"""Copy the outputs of tools/final_runs.sh from gpurun_out/ into profiles/ (bench lines, GPU suite
tail, launch list + summary), regenerate profiles/r2_ncu_stream.md and the cfg3 / cfg4 entries of
profiles/traffic.json from the two ncu --set full reports, and print the table DESIGN.md section 5 quotes.
usage: python tools/collect_final.py"""
import json
import re
import shutil
import subprocess

G, P = "gpurun_out/", "profiles/"
for c in range(5):
    shutil.copy(f"{G}final_cfg{c}.json", f"{P}r2_final_cfg{c}.json")
shutil.copy(G + "final_cfg3_fp32.json", P + "r2_final_cfg3_fp32.json")
shutil.copy(G + "final_ref_cfg3.json", P + "r2_final_ref_cfg3.json")
shutil.copy(G + "final_gputests.txt", P + "r2_final_gputests.txt")
shutil.copy(G + "final_launches.csv", P + "r2_cfg3_launches.csv")
open(P + "r2_cfg3_launches_summary.txt", "w").write(
    subprocess.run(["python", "tools/launch_summary.py", P + "r2_cfg3_launches.csv"], capture_output=True, text=True).stdout)


def summ(rep, k):
    return subprocess.run(["python", "tools/ncu_summary.py", rep, k], capture_output=True, text=True).stdout


def dram(txt):
    mul = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    r = re.search(r"dram__bytes_read.sum\s+([\d.]+) (\w+)", txt)
    w = re.search(r"dram__bytes_write.sum\s+([\d.]+) (\w+)", txt)
    return int(float(r.group(1)) * mul[r.group(2)] + float(w.group(1)) * mul[w.group(2)])


out = ["# Round 2 ncu captures of the stream encode (final build)", "",
       "Commands: `tools/prof_embed.sh final` under gpurun, one B200: launch list of a 3-step configs[3] bench",
       "(`profiles/r2_cfg3_launches.csv`, summary `r2_cfg3_launches_summary.txt`), then `ncu --set full --clock-control none --import-source on`",
       "of one encode of configs[3] (every k_st_* pass) and of k_st_embed at configs[4] (`tools/encode_once.py`).",
       "Cold clean L2 per launch (ncu replay), so absolute times differ slightly from the bench's live per-kernel times.",
       "The shared-memory pipe analysis of k_st_embed (session 4, before / after the conflict-free factor pass) is in",
       "`profiles/r2_s4_embed_l1.md`.", ""]
traffic = {}
for k in ["k_st_embed", "k_st_part1", "k_st_part2", "k_st_degree", "k_st_hist2", "k_st_hist1"]:
    t = summ(G + "final_full_c3.ncu-rep", k)
    out += [f"## {k}, configs[3]", "```", t.rstrip(), "```"]
    traffic[k] = dram(t)
t = summ(G + "final_full_c4.ncu-rep", "k_st_embed")
out += ["## k_st_embed, configs[4]", "```", t.rstrip(), "```"]
lines = subprocess.run(["python", "tools/ncu_smem_lines.py", G + "final_full_c3.ncu-rep", "k_st_embed", "10"],
                       capture_output=True, text=True).stdout
out += ["## k_st_embed, configs[3]: shared-memory (L1) wavefronts by source line (tools/ncu_smem_lines.py)",
        "(the atomicAdd row appears twice: the call site and the inlined CAS loop are the same instructions)",
        "```", lines.rstrip(), "```"]
open(P + "r2_ncu_stream.md", "w").write("\n".join(out) + "\n")
tj = json.load(open(P + "traffic.json"))
tj["cfg3"], tj["cfg4"] = traffic, {"k_st_embed": dram(t)}
json.dump(tj, open(P + "traffic.json", "w"), indent=1)

for c in range(5):
    d = [json.loads(x) for x in open(f"{P}r2_final_cfg{c}.json") if x.startswith("{")][-1]
    ks = " ".join(f"{k['kernel']}={k['ms_per_launch']:.3f}" for k in d["kernels"][:7])
    print(f"cfg{c}: {d['value'] / 1e9:.2f} G edges/s, {d['ms_per_step']:.3f} ms, {d['roofline']['kernel']} "
          f"{d['roofline']['frac']:.3f}, e2e {d['e2e']['value'] / 1e9:.3f} G/s, cpu {d['cpu_baseline']['value'] / 1e6:.2f} M/s | {ks}")
d = [json.loads(x) for x in open(P + "r2_final_cfg3_fp32.json") if x.startswith("{")][-1]
print(f"cfg3 fp32: {d['value'] / 1e9:.2f} G edges/s, {d['ms_per_step']:.3f} ms, embed frac {d['embed_kernel']['frac']:.3f}, "
      f"e2e {d['e2e']['value'] / 1e9:.3f}")
d = [json.loads(x) for x in open(P + "r2_final_ref_cfg3.json") if x.startswith("{")][-1]
print(f"reference arm: {d['value'] / 1e6:.2f} M edges/s, {d['ms_per_step'] / 1e3:.1f} s per run, {d['steps']} runs")
print(open(P + "r2_final_gputests.txt").read().strip().splitlines()[-1])
