"""tsbench (cmd: route) argument handling without a GPU."""

import subprocess
import sys


def test_invalid_config_reports_status():
    p = subprocess.run([sys.executable, "-m", "paper_2407_11488_b200.tsbench", "--kernel", "hotspot",
                        "--config", "1024,32,10,10,10,10,1"], capture_output=True, text=True)
    assert p.returncode != 0 and "TUNE_STATUS invalid" in p.stdout
