"""bench.py contract on CPU: the --gpus N launch (N ranks over gloo, max-over-ranks time,
summed points) and the reference arm (the reference's own oracle on the host cores,
without the B200 library)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _last_json(out: str) -> dict:
    return json.loads([ln for ln in out.strip().splitlines() if ln.startswith("{")][-1])


def test_gpus_n_launches_n_ranks_and_takes_the_max():
    env = dict(os.environ, HF_BENCH_SELFTEST="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "5",
                        "--warmup", "3", "--workload", "config5", "--scaling", "strong"],
                       capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _last_json(r.stdout)
    assert line["selftest"] is True and line["n_gpus"] == 2
    assert line["points_all"] == 1000 + 2000            # summed over both ranks
    assert line["ms_per_step"] >= 19.0                   # rank 1 sleeps 20 ms per step: the max wins
    assert line["ms_per_step"] > line["rank0_ms_per_step"] * 1.5
    assert line["config"] == bench.workload_config("config5", 2, "strong")
    assert line["config"]["parallelism"].startswith("element-partition x2")


def test_workload_config_is_device_free_and_scales():
    c1 = bench.workload_config("config5", 1, "weak")
    assert c1["points_per_step"] == sum(bench.case_elements(d, p, pr, t)[1] * (p + 1) ** d
                                        for d, p, pr, t in bench.workload_cases("config5"))
    assert bench.workload_config("config5", 4, "weak")["points_per_step"] == 4 * c1["points_per_step"]
    assert bench.workload_config("config5", 4, "strong")["points_per_step"] == c1["points_per_step"]
    # config 5: 1.5e8 points per case, 2,343,750 / 694,444 elements, rounded to
    # whole groups of the selected chunk (p3 FP64: 4 elements)
    g3, n3 = bench.case_elements(3, 3, "fp64", 1.5e8)
    assert n3 % g3 == 0 and abs(n3 - 2343750) < g3
    assert abs(bench.case_elements(3, 5, "fp64", 1.5e8)[1] - 694445) <= 1


def test_every_workload_case_has_a_static_group():
    for w in bench.WORKLOAD_DESC:
        for d, p, prec, _ in bench.workload_cases(w):
            assert (d, p, prec) in bench.GPU_GROUPS


def test_cpu_sample_is_proportional_and_group_aligned():
    s = bench.cpu_sample_cases("config3", 1e6)
    for d, p, prec, g, n in s:
        assert n % g == 0 and n >= g
    pts = [n * (p + 1) ** d for d, p, _, _, n in s]
    assert pts[-1] > 5 * pts[0]                           # d2 p8 carries ~20x the points of p1


def test_reference_arm_runs_without_the_b200_library():
    probe = (
        "import sys, runpy, json\n"
        f"sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '3', '--ref-budget', '2e5']\n"
        f"runpy.run_path({os.path.join(ROOT, 'bench.py')!r}, run_name='__main__')\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'b200_loaded': 'libhexfuse_b200' in maps,\n"
        "                  'oracle_restatement_loaded': 'libhexfuse_oracle.so' in maps,\n"
        "                  'torch_imported': 'torch' in sys.modules,\n"
        "                  'package_imported': any(m.startswith('paper_2107_14027_b200') for m in sys.modules)}))\n")
    r = subprocess.run([sys.executable, "-c", probe], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(ln) for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    ref, probe_out = lines[-2], lines[-1]
    assert probe_out == {"b200_loaded": False, "oracle_restatement_loaded": False, "torch_imported": False,
                         "package_imported": False}
    assert ref["impl"] == "reference" and ref["value"] > 0
    assert ref["config"] == bench.workload_config("config2", 1, "weak")
    cb = ref["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and "-march" in cb["build"]
    assert ref["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_two_rank_bench_on_one_gpu():
    """The N-rank path of bench.py (re-launch under torch.distributed.run, element partition,
    max-over-ranks timing, sums of points) with real kernels: two ranks sharing the box's GPU
    (HF_BENCH_SHARED_GPU: reductions over gloo); weak and strong config 5 partition."""
    env = dict(os.environ, HF_BENCH_SHARED_GPU="1")
    for extra, scaling in (([], "weak"), (["--workload", "config5", "--scaling", "strong"], "strong")):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                            "--warmup", "3", "--no-cpu", "--no-e2e"] + (extra or ["--workload", "config1"]),
                           capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
        assert r.returncode == 0, r.stderr[-3000:]
        line = json.loads(r.stdout.strip().splitlines()[-1])
        assert line["n_gpus"] == 2 and line["scaling"] == scaling and line["value"] > 0
        assert line["parity"]["ok"]
        want = bench.workload_config(line["config"]["workload"], 2, scaling)["points_per_step"]
        assert line["config"]["points_per_step"] == want
