python -m pytest tests -m gpu -q (device guards on handles)
