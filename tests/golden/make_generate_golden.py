"""Regenerate the `flowpipe generate` CSV fixtures from the UNMODIFIED reference
(run in the build container, where /root/reference exists):

    python tests/golden/make_generate_golden.py

Each case is one `python -m flowpipe generate ...` invocation; the CSV bytes are
stored under tests/golden/generate/ for tests/test_gpu_output.py."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = {
    "n3_s4_seed123": ["--num-images", "3", "--steps", "4", "--seed", "123"],
    "n4_s4_seed123": ["--num-images", "4", "--steps", "4", "--seed", "123"],
    "n5_s2_seed7_w7.5": ["--num-images", "5", "--steps", "2", "--seed", "7", "--guidance", "7.5"],
    "n2_s8_seed0_compiled": ["--num-images", "2", "--steps", "8", "--seed", "0", "--engine", "compiled"],
}

if __name__ == "__main__":
    env = dict(os.environ, PYTHONPATH="/root/reference/pkg/src")
    os.makedirs(os.path.join(HERE, "generate"), exist_ok=True)
    for name, args in CASES.items():
        out = os.path.join(HERE, "generate", f"{name}.csv")
        subprocess.run([sys.executable, "-m", "flowpipe", "generate", *args, "--out", out], env=env, check=True,
                       cwd="/tmp")
        print(name, os.path.getsize(out))
