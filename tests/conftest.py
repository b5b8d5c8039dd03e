import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: longer CPU test")


def run_group(cmd, timeout=300, env=None, cwd=None):
    """Run a multi-process launcher (torchrun) in its own process group and, if it
    does not finish within `timeout` seconds, kill that whole group (the launcher AND
    its rank processes): a hung rank must not outlive its test and keep spinning on the
    GPUs that later tests and benches use.  Returns a CompletedProcess (rc -9 on a
    timeout, with the timeout noted in stderr)."""
    import os
    import signal
    import subprocess
    p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, cwd=cwd, env=env,
                         start_new_session=True)
    try:
        out, err = p.communicate(timeout=timeout)
        return subprocess.CompletedProcess(cmd, p.returncode, out, err)
    except subprocess.TimeoutExpired:
        # SIGTERM first: torchrun's handler terminates its rank processes (each in a
        # session of its own); then SIGKILL whatever is left of the group we created
        for sig, wait in ((signal.SIGTERM, 60), (signal.SIGKILL, None)):
            try:
                os.killpg(p.pid, sig)
            except ProcessLookupError:
                break
            try:
                out, err = p.communicate(timeout=wait)
                break
            except subprocess.TimeoutExpired:
                continue
        out, err = p.communicate()
        return subprocess.CompletedProcess(cmd, -9, out, (err or "") + f"\n[run_group] killed after {timeout} s")
