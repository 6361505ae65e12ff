#!/bin/bash
# Install the UNMODIFIED reference (tunescape, pure Python) under baseline/_ref.
# Its build writes into the source tree, so it installs from a copy; its
# dependencies (numpy, scipy, PyYAML, click) are already in the image, hence
# --no-deps (dependency resolution against the offline wheelhouse fails).
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/tunescape_src baseline/_ref
cp -r /root/reference/pkg /tmp/tunescape_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref /tmp/tunescape_src
make -s -C oracle tsbench_cpu
echo "installed: $(ls baseline/_ref)"
