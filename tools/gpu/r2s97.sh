python -m pytest tests -m gpu -q; smoke (final code)
