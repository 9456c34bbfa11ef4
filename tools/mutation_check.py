"""Mutation check of the GPU parity suite (run on a GPU box): each mutation plants one plausible mistake in
a copy of the repo (a dropped ReLU mask, a one-sided error clip, a missing terminal select, a skipped target
refresh, r updated after theta, a store instead of an accumulate, a fetch of a stale generation), rebuilds
libdqn.so there and runs the parity tests that must catch it. A mutation that the listed tests still pass is
a hole in the suite.

usage: python tools/mutation_check.py [--only NAME] > gpurun_out/mutations.txt
"""
import argparse
import os
import shutil
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = "paper_1508_04186_b200/csrc/"
B16 = CSRC + "kernels_bf16.cu"
G = "tests/test_gpu_parity_gated.py::"

# name: ([(file, exact text, replacement), ...], pytest node ids of which at least one must fail)
MUTATIONS = {
    "head_dH_relu_mask": ([(CSRC + "kernels_head.cu", "const float d = s_h0[u] > 0.0f ? dq * s_wa[u] : 0.0f;",
                            "const float d = dq * s_wa[u];")], [G + "test_gated_one_step[mnih-b32]"]),
    "fc_dX_relu_mask": ([(B16, "(mk[i] & 0x8000u) == 0 && mk[i] != 0 ? v[i] : 0.0f", "v[i]")],
                        [G + "test_gated_one_step[mnih-b32]"]),
    "conv1_dZ_relu_mask_even_channels": ([(B16, "const float d_lo = a_lo > 0.0f ? v[16 * q + 2 * h] : 0.0f;",
                                           "const float d_lo = v[16 * q + 2 * h];")],
                                         [G + "test_gated_one_step[mnih-b32]"]),
    "conv1_dZ_relu_mask": ([(B16, "const float d_lo = a_lo > 0.0f ? v[16 * q + 2 * h] : 0.0f;",
                             "const float d_lo = v[16 * q + 2 * h];"),
                            (B16, "const float d_hi = a_hi > 0.0f ? v[16 * q + 2 * h + 1] : 0.0f;",
                             "const float d_hi = v[16 * q + 2 * h + 1];")], [G + "test_gated_one_step[mnih-b32]"]),
    "tconv_dgrad_relu_mask": ([(CSRC + "kernels_tma.cu",
                                "const __nv_bfloat162 h2 = __floats2bfloat162_rn(bf16_gt0(mw[h] & 0xFFFFu) ? v[2 * h] : 0.0f,\n"
                                "                                                            bf16_gt0(mw[h] >> 16) ? v[2 * h + 1] : 0.0f);",
                                "const __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * h], v[2 * h + 1]);")],
                              [G + "test_gated_one_step[scaled-b32]"]),
    "tgemm_fc_dX_relu_mask": ([(CSRC + "kernels_tma.cu", "__float2bfloat16_rn(bf16_gt0(mk[i]) ? v[i] : 0.0f)",
                                "__float2bfloat16_rn(v[i])")], [G + "test_gated_one_step[scaled-b32]"]),
    "twgrad_tap_shift_dropped": ([(CSRC + "kernels_tma.cu",
                                   "off[k][hh] = cb * win_bytes(a.R) + ((t / a.Tw) * a.Ws + t % a.Tw) * 128;",
                                   "off[k][hh] = cb * win_bytes(a.R);")],
                                      [G + "test_gated_one_step[scaled-b32]"]),
    "error_clip_one_sided": ([(CSRC + "kernels_head.cu", "dc = fminf(fmaxf(dc, -h.clip), h.clip);",
                               "dc = fminf(dc, h.clip);")], [G + "test_gated_error_clip[mnih]"]),
    "terminal_select_dropped": ([(CSRC + "kernels_head.cu", "const float y = term ? r : r + h.gamma * best;",
                                  "const float y = r + h.gamma * best;")], [G + "test_gated_one_step[mnih-b32]"]),
    "target_refresh_bf16_skipped": ([(
        CSRC + "dqn_runtime.cu",
        "    CK(cudaMemcpyAsync(ctx->theta_hat_bf16, ctx->theta_local_bf16, sizeof(__nv_bfloat16) * ctx->P_bf16,\n"
        "                       cudaMemcpyDeviceToDevice, st));\n    PE();\n  }\n  // a1-a4: sample",
        "    PE();\n  }\n  // a1-a4: sample")], [G + "test_target_refresh_and_bf16_working_copies[mnih]"]),
    "rmsprop_theta_uses_old_r": ([
        (B16, "  const float rr = __fmaf_rn(u.rho, r, __fmul_rn(__fmul_rn(u.omr, gb), gb));",
         "  const float r0 = r;\n  const float rr = __fmaf_rn(u.rho, r, __fmul_rn(__fmul_rn(u.omr, gb), gb));"),
        (B16, "th = __fmaf_rn(-__fmul_rn(u.lr, gb), rsqrtf(__fadd_rn(rr, u.eps)), th);",
         "th = __fmaf_rn(-__fmul_rn(u.lr, gb), rsqrtf(__fadd_rn(r0, u.eps)), th);")],
        [G + "test_gated_k_steps_delta_theta[mnih]"]),
    "fc_dW_store_not_accumulate": ([(CSRC + "dqn_runtime.cu", "  gw.store = c.n_push == 1;", "  gw.store = 1;")],
                                   [G + "test_gated_accumulate_n_push3"]),
    "async_fetch_one_generation_older": ([(
        CSRC + "kernels_comm.cu", "const long long m = forced >= 0 ? forced : (long long)g;",
        "const long long m = forced >= 0 ? forced : (long long)g - (g > 0 ? 1 : 0);")],
        ["tests/test_gpu_async.py::test_async_free_running_fp32_equals_its_realised_schedule[4-1-2-0]"]),
    "prio_sqrt_dropped": ([(CSRC + "kernels_prio.cu", "    if (alpha_half) p = __fsqrt_rn(p);\n", "")],
                          ["tests/test_gpu_prio.py::test_prioritized_replay_teacher_forced[fp32-a05]"]),
    "prio_max_priority_not_kept": ([(CSRC + "kernels_prio.cu", "    *maxp = mm;\n", "")],
                                   ["tests/test_gpu_prio.py::test_prioritized_replay_teacher_forced[fp32-a1]"]),
    "prio_not_stratified": ([(CSRC + "kernels_prio.cu", "float r = __fmul_rn(__fadd_rn((float)j, u), __fdiv_rn(S, (float)b));",
                              "float r = __fmul_rn(u, S);")],
                            ["tests/test_gpu_prio.py::test_prioritized_replay_teacher_forced[fp32-a1]"]),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    names = [a.only] if a.only else list(MUTATIONS)
    base = "/tmp/dqn_mut"
    results = []
    for name in names:
        edits, tests = MUTATIONS[name]
        work = os.path.join(base, name)
        shutil.rmtree(work, ignore_errors=True)
        shutil.copytree(ROOT, work, ignore=shutil.ignore_patterns(".git", "gpurun_out", "build", "*.so", "__pycache__"))
        for ff, o, n in edits:
            p = os.path.join(work, ff)
            src = open(p).read()
            assert src.count(o) == 1, f"{name}: anchor not found exactly once in {ff}"
            open(p, "w").write(src.replace(o, n))
        t0 = time.time()
        b = subprocess.run([sys.executable, "-c", "from paper_1508_04186_b200 import build as B; B.build(force=True)"],
                           cwd=work, capture_output=True, text=True)
        if b.returncode != 0:
            results.append((name, "BUILD FAILED", b.stderr[-500:]))
            print(f"{name}: BUILD FAILED", flush=True)
            continue
        # the oracle is test infrastructure: reuse the unmutated build
        shutil.copy(os.path.join(ROOT, "oracle", "liboracle.so"), os.path.join(work, "oracle", "liboracle.so"))
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *tests], cwd=work,
                           capture_output=True, text=True, timeout=1200)
        caught = r.returncode != 0
        last = [ln for ln in r.stdout.splitlines() if "passed" in ln or "failed" in ln or "Error" in ln][-1:]
        results.append((name, "CAUGHT" if caught else "MISSED",
                        f"{' '.join(tests)} -> {last} ({time.time() - t0:.0f} s)"))
        print(f"{name}: {results[-1][1]}  {results[-1][2]}", flush=True)
        shutil.rmtree(work, ignore_errors=True)
    missed = [r for r in results if r[1] != "CAUGHT"]
    print(f"\n{len(results) - len(missed)} of {len(results)} mutations caught", flush=True)
    sys.exit(1 if missed else 0)


if __name__ == "__main__":
    main()
