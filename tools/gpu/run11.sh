set -x
timeout 900 python tools/profile_step.py --config pix2pix --batch 1 --incore 2>&1 | head -45
timeout 900 python tools/profile_step.py --config deeplab --batch 4 --incore 2>&1 | head -45
